"""PCIe probe: pinned H2D / D2H bandwidth alone, concurrently, and D2H split over 2 streams
(context for the e2e number of bench.py; not part of the product)."""
import json
import torch

GB = 1 << 30
h_in = torch.empty(int(1.1e9), dtype=torch.uint8).pin_memory()
d_in = torch.empty_like(h_in, device="cuda")
h_out = torch.empty(int(3.46e9), dtype=torch.uint8).pin_memory()
d_out = torch.empty_like(h_out, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        for s in (s1, s2, s3):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def d2h_split():
    half = h_out.numel() // 2
    with torch.cuda.stream(s2):
        h_out[:half].copy_(d_out[:half], non_blocking=True)
    with torch.cuda.stream(s3):
        h_out[half:].copy_(d_out[half:], non_blocking=True)


def both():
    h2d()
    d2h()


r = {}
for name, fn, nbytes in (("h2d", h2d, h_in.numel()), ("d2h", d2h, h_out.numel()), ("d2h_split2", d2h_split, h_out.numel()),
                         ("both", both, h_in.numel() + h_out.numel())):
    ms = timed(fn)
    r[name] = {"ms": round(ms, 2), "GB/s": round(nbytes / ms / 1e6, 1)}
print(json.dumps(r))
