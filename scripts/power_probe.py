"""Per-launch decode time over a long run (eager launches, events around each) with NVML
SM / memory clocks, power and throttle reasons sampled alongside: does the kernel slow
down after the first tens of milliseconds (power / thermal management)?

    python scripts/power_probe.py [--launches 400] [--instances 1000]
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=400)
    ap.add_argument("--instances", type=int, default=1000)
    args = ap.parse_args()
    import pynvml
    import torch
    import bench
    import paper_2404_06359_b200 as mc
    torch.cuda.set_device(0)
    blob, _ = bench.build_blob(mc, "cfg4_city", 0, 1, 2, args.instances)
    db = mc.DeviceBlob(blob, want_vertices=True)
    for _ in range(5):
        db.decode()
    torch.cuda.synchronize()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def poll():
        t0 = time.perf_counter()
        while not stop.is_set():
            try:
                samples.append((time.perf_counter() - t0, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                                pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.002)

    th = threading.Thread(target=poll, daemon=True)
    th.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.launches)]
    for a, b in ev:
        a.record()
        db.decode()
        b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    out = {"launches": args.launches, "instances": args.instances,
           "ms_by_block_of_25": [round(float(x), 4) for x in ms.reshape(-1, 25).mean(1)] if args.launches % 25 == 0 else None,
           "ms_first10": [round(float(x), 4) for x in ms[:10]], "ms_median": float(np.median(ms)),
           "samples": [(round(t, 3), s, m, round(p, 1), r) for t, s, m, p, r in samples[::5]]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
