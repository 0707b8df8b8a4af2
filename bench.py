#!/usr/bin/env python
"""Benchmark: per-meshlet decompression (arXiv 2404.06359) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4_city] [--impl ours|reference]

One STEP = one decode of the rank's whole shard of the scene (every §8(a) row:
record staging, index expansion, L/R lookback, triangle assembly, attribute unpack +
dequantisation, index and vertex stores) = one launch of the sm_100a kernel.

Default workload (N=1): BASELINE cfg4, the instanced synthetic city, 1000 instances of
16 seeded buildings x 99,372 tris = 99.4M triangles per GPU, 64v/126t meshlets,
GTS-Reuse, pos3 + oct2 + uv2 at 16 bits.  At N>1 every rank decodes its own
1000-instance shard of an N x 1000-instance city (weak scaling; no data-path
collective; one NCCL all-reduce of the checksum after timing).

Inputs (~1 GB compressed) and outputs (~3.6 GB) are far larger than the 126 MB L2, so
no L2 flush is needed between steps; the smaller parity workloads (--workload cfg1-3,
working set < 4 x L2) flush L2 between steps and time the sum of the launches.  Timing:
CUDA events on the launching stream, barrier + synchronize on both sides, max over ranks.

Prints ONE JSON line on rank 0.  ``--impl reference`` times the oracle (plain-C
sequential decoder, ``oracle/``) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "decoded triangles/sec (HBM GB/s vs B200 peak in roofline)"
CODEC_NAMES = {1: "gts", 2: "gts-reuse", 3: "basic"}
UNIT = "Gtri/s"

L2_BYTES = 126 * 1000 * 1000   # B200 L2 (B200_PROFILING.md)

WORKLOADS = {
    "cfg1_grid": dict(desc="32x32 quad grid, 2,048 tris, pos3+nrm3+uv2 @16b", vmax=64, tmax=126),
    "cfg2_torus": dict(desc="torus 1000x500, 1M tris, pos3 @16b", vmax=64, tmax=126),
    "cfg3_sphere": dict(desc="displaced cube-sphere 12*913^2 = 10.0M tris, pos3+oct2+uv2 @16b", vmax=64, tmax=126),
    "cfg4_city": dict(desc="instanced city, 1000 instances x 99,372 tris per GPU, pos3+oct2+uv2 @16b",
                      vmax=64, tmax=126),
    "cfg3_sphere_nrm8": dict(desc="cfg3 sphere with raw normals: pos3+nrm3+uv2 @16b (the paper's 8 attributes)",
                             vmax=64, tmax=126),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- scenes

def build_blob(mc, workload: str, rank: int, world: int, codec: int, instances: int, protos_k=(16, 91),
               vw: bool = False, cull: bool = False):
    """The rank's shard of the workload as a product-encoded blob (mc_encode path)."""
    w = WORKLOADS[workload]
    if workload == "cfg4_city":
        scene = synth.city(num_instances=instances * world, num_prototypes=protos_k[0], k=protos_k[1], seed=0)
        protos = [mc.mc_encode(p, w["vmax"], w["tmax"], codec, variable_widths=vw, cull_cones=cull)
                  for p in scene.prototypes]
        blob = mc.mc_blob_instance_range(protos, scene.instance_proto, scene.instance_offset,
                                         rank * instances, instances)
        meta = {"instances_per_gpu": instances, "prototypes": protos_k[0],
                "restarts_per_meshlet": round(sum(p.encode_stats()["restarts"] for p in protos) /
                                              max(1, sum(p.layout.num_meshlets for p in protos)), 3)}
        return blob, meta
    mesh = {"cfg1_grid": lambda: synth.quad_grid(32, 32),
            "cfg2_torus": lambda: synth.torus(1000, 500),
            "cfg3_sphere": lambda: synth.displaced_sphere(913),
            "cfg3_sphere_nrm8": lambda: synth.displaced_sphere(913, oct_normals=False)}[workload]()
    blob = mc.mc_encode(mesh, w["vmax"], w["tmax"], codec, variable_widths=vw, cull_cones=cull)
    meta = {"restarts_per_meshlet": round(blob.encode_stats()["restarts"] / max(1, blob.layout.num_meshlets), 3)}
    if world > 1:   # strong-sharded replicas of the single mesh
        f, c = blob.shard_ranges(world)[rank]
        blob = blob.extract(f, c)
    return blob, meta


def record_real_triangles(data: np.ndarray, m0: int, m1: int) -> int:
    """Σ T = T' - 4R over records [m0, m1) read straight from FORMAT.md bytes."""
    off_dir = int(data[64:72].view(np.uint64)[0])
    off_rec = int(data[80:88].view(np.uint64)[0])
    M = int(data[16:20].view(np.uint32)[0])
    d = data[off_dir:off_dir + 4 * (M + 1)].view(np.uint32)[m0:m1].astype(np.int64) * 16 + off_rec
    tp = data[d + 9].astype(np.int64) + 1
    r = data[d + 12].astype(np.int64) | (data[d + 13].astype(np.int64) << 8)
    return int((tp - 4 * r).sum())


def allreduce_u64_sum(values, dist, device):
    """All-reduce u64 checksums (FORMAT.md §6): int64 sum wraps mod 2^64 exactly like u64."""
    import torch
    t = torch.tensor(np.array(values, dtype=np.uint64).view(np.int64), device=device)
    if dist is not None:
        dist.all_reduce(t)
    return [int(x) for x in t.cpu().numpy().view(np.uint64)]


# ----------------------------------------------------------------------------- oracle timing (CPU)

def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_time(data: np.ndarray, seconds: float, cores: int):
    """Time the oracle decoder (as it stands) on `cores` host threads: passes over the
    first S records (S calibrated so one pass takes about `seconds`, capped at the whole
    workload), repeated until at least `seconds` of wall time have elapsed.
    Returns (tri/s, S, T, wall, passes) with T the real triangles decoded over all passes."""
    import oracle
    info = oracle.blob_info(data)
    M = info.M

    # calibrate on one thread
    cal = min(M, 400)
    tp_cal = 3 * 256 * cal
    idx = np.zeros(tp_cal, np.uint32)
    q = None
    f = np.zeros(info.n_out * 256 * cal, np.float32)
    t0 = time.perf_counter()
    oracle.decode_range_raw(data, 0, cal, idx, q, f)
    per_rec = (time.perf_counter() - t0) / max(cal, 1)
    S = int(min(M, max(cal, seconds * cores / max(per_rec, 1e-9))))
    # output buffers sized for records [0, S)
    tot_tp = 3 * 256 * S if S < M else 3 * info.total_tp
    tot_v = 256 * S if S < M else info.total_v
    idx = np.zeros(min(tot_tp, 3 * info.total_tp), np.uint32)
    f = np.zeros(info.n_out * min(tot_v, info.total_v), np.float32)
    bounds = np.linspace(0, S, cores * 4 + 1).astype(np.int64)
    T1 = record_real_triangles(data, 0, S)
    passes = 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        while True:
            list(ex.map(lambda i: oracle.decode_range_raw(data, int(bounds[i]), int(bounds[i + 1]), idx, None, f),
                        range(len(bounds) - 1)))
            passes += 1
            if time.perf_counter() - t0 >= seconds or passes >= 10000:
                break
    wall = time.perf_counter() - t0
    T = T1 * passes
    return T / wall, S, T, wall, passes


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """Polls NVML SM clock and throttle reasons during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, torch, dev):
        self.ok = False
        self.samples, self.reasons = [], set()
        try:
            import pynvml
            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(dev)
            h = None
            try:
                bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("LOCAL_RANK", dev)))
            self.nv, self.h = pynvml, h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": int(self.max_mhz),
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        return json.load(open(p))[workload]["dram_bytes_per_launch"]
    except Exception:
        return None


# ----------------------------------------------------------------------------- arms

def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, on host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    import paper_2404_06359_b200 as mc
    blob, meta = build_blob(mc, args.workload, 0, 1, args.codec, args.instances, vw=args.variable_widths)
    data = np.array(blob.bytes)
    cores = host_cores()
    per_step = max(0.5, min(3.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_time(data, min(per_step, 1.0), cores)
    rates, walls, tris, recs = [], [], 0, 0
    for _ in range(args.steps):
        r, S, T, wall, passes = oracle_time(data, per_step, cores)
        rates.append(r)
        walls.append(wall)
        tris += T
        recs = S
    value = tris / sum(walls) / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/fp32",
            "data": "synthetic", "config": {"workload": args.workload, **WORKLOADS[args.workload], **meta},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"per step: {passes} pass(es) over the first {recs} records of the workload "
                                       f"(>= {per_step:.1f}s of CPU work)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2404_06359_b200 as mc
    mc.lib()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    t0 = time.time()
    blob, meta = build_blob(mc, args.workload, rank, world, args.codec, args.instances, vw=args.variable_widths,
                            cull=args.cull)
    L = blob.layout
    log(f"[rank {rank}] scene built in {time.time() - t0:.1f}s: {L.num_meshlets} meshlets, "
        f"T={L.total_t} T'={L.total_tp} V={L.total_v}, {L.total_bytes / 1e6:.1f} MB")
    db = mc.DeviceBlob(blob, device=dev, want_vertices=True, want_quantized=False, index_format=args.index_format)
    stream = torch.cuda.current_stream(dev)
    alg_bytes = db.algorithmic_bytes()
    view_dir = np.array([1.0, 2.0, -3.0], np.float64)
    view_dir = (view_dir / np.linalg.norm(view_dir)).astype(np.float32)
    if args.cull:   # FORMAT.md §7: one step = cull + scan + emit + decode of the visible records
        step = lambda: db.decode_culled(view_dir, stream=stream)
        launches_per_step = 4
    else:
        step = lambda: db.decode(stream=stream)
        launches_per_step = 1

    # ---------------- device-resident timing (the headline `value`)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # working sets under 4 x L2 (cfg1-cfg3) would be partly L2-resident from the previous
    # step: flush L2 between steps by writing a 2 x L2 buffer, outside the per-launch events,
    # and time the sum of the launches; cfg4 (4.6 GB per step) needs no flush
    flush = alg_bytes < 4 * L2_BYTES
    fbuf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev) if flush else None
    with ClockSampler(torch, dev) as clk:
        g0.record(stream)
        for k in range(args.steps):
            if flush:
                fbuf.zero_()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        g1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launch_ms = np.array([a.elapsed_time(b) for a, b in ev])
    total_ms = float(launch_ms.sum()) if flush else g0.elapsed_time(g1)
    tri_local = L.total_t
    t = torch.tensor([total_ms, float(launch_ms.mean())], dtype=torch.float64, device=dev)
    n = torch.tensor([float(tri_local), float(alg_bytes)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
    max_ms, max_launch_ms = float(t[0]), float(t[1])
    tri_all, bytes_all = float(n[0]), float(n[1])
    value = tri_all * args.steps / (max_ms * 1e-3) / 1e9

    cull_info = None
    if args.cull:
        cc = db.read_cull_counts()
        vis_bytes = int(alg_bytes * cc["Tp"] / max(1, L.total_tp))   # approx: bytes scale with decoded work
        cull_info = {"view_dir": [float(x) for x in view_dir], "visible_records": cc["records"],
                     "visible_fraction_records": cc["records"] / max(1, L.num_meshlets),
                     "visible_triangles": cc["T"], "visible_decoded_triangles": cc["Tp"],
                     "visible_gtri_s": cc["T"] * args.steps * world / (max_ms * 1e-3) / 1e9,
                     "value_counts": "all scene triangles (culled ones included) per second"}
        alg_bytes = vis_bytes
    # ---------------- verification after timing: checksum all-reduce (the only collective)
    st = db.decode_culled(view_dir, stream=stream, stats=True) if args.cull else db.decode_stats(stream=stream)
    checksum = allreduce_u64_sum([st["checksum_indices"], st["checksum_vertices"]], dist, dev)
    errs = torch.tensor([st["error_bits"]], dtype=torch.int64, device=dev)
    if dist:
        dist.all_reduce(errs)

    # ---------------- end to end through the C ABI with pinned HOST buffers
    e2e = None
    if not args.no_e2e and not args.cull:
        data = np.array(blob.bytes)
        h_blob = torch.from_numpy(data).pin_memory()
        idx_words = (1 if args.index_format == "u8x4" else 3) * L.total_tp
        h_idx = torch.empty(idx_words, dtype=torch.int32).pin_memory()
        h_v = torch.empty(L.n_out * L.total_v, dtype=torch.float32).pin_memory()
        ke = max(1, min(args.steps, args.e2e_steps))
        for _ in range(1):
            mc.mc_decode_host(L, h_blob, db.d_blob, h_idx, db.indices, h_v, db.vertices, flags=db.index_flags,
                              stream=stream, chunks=args.e2e_chunks)
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            mc.mc_decode_host(L, h_blob, db.d_blob, h_idx, db.indices, h_v, db.vertices, flags=db.index_flags,
                              stream=stream, chunks=args.e2e_chunks)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": tri_all * ke / (float(et[0]) * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(data.nbytes), "d2h_bytes_per_step": int(4 * idx_words + 4 * L.n_out * L.total_v),
               "steps": ke, "chunks": args.e2e_chunks,
               "path": "mc_decode_host (pinned host blob -> HBM -> decode -> pinned host outputs; "
                       "chunks >= 2: H2D / decode / D2H pipelined over record ranges)"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_src = peak_hbm()
    achieved = alg_bytes / (max_launch_ms * 1e-3) / 1e9
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle
        oracle.build()
        cores = host_cores()
        rate, S, T, wall, passes = oracle_time(np.array(blob.bytes), args.cpu_seconds, cores)
        cpu = {"value": rate / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{passes} pass(es) over the first {S} of {L.num_meshlets} records "
                         f"({T} tris decoded in total), {wall:.1f}s wall on {cores} threads"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32/fp32", "data": "synthetic",
        "config": {"workload": args.workload, "desc": WORKLOADS[args.workload]["desc"],
                   "codec": CODEC_NAMES[args.codec], "index_format": args.index_format,
                   "attribute_widths": "per-meshlet (VW)" if args.variable_widths else "global b",
                   "compressed_bits_per_tri": round(8.0 * L.total_bytes / max(1, L.total_t), 3),
                   "meshlet": f"{WORKLOADS[args.workload]['vmax']}v/{WORKLOADS[args.workload]['tmax']}t",
                   "triangles_per_gpu": int(tri_local), "decoded_triangles_incl_degenerate_per_gpu": int(L.total_tp),
                   "meshlets_per_gpu": int(L.num_meshlets), "compressed_bytes_per_gpu": int(L.total_bytes),
                   "l2": (f"L2 flushed between steps ({2 * L2_BYTES >> 20} MiB memset, outside the timed launches; "
                          f"working set {alg_bytes / 1e6:.0f} MB < 4 x L2); value from the summed per-launch events")
                   if flush else f"inputs+outputs ({alg_bytes / 1e9:.2f} GB) >> 126 MB L2 each step (no flush)", **meta},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(args.workload), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": int(alg_bytes),
                     "launch_ms": max_launch_ms},
        "hbm_gbs_aggregate": bytes_all * args.steps / (max_ms * 1e-3) / 1e9,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps * launches_per_step,
        "cull": cull_info,
        "clocks": clk.summary(),
        "checksum": {"indices": checksum[0], "vertices": checksum[1], "error_bits": int(errs.item())},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=list(WORKLOADS), default="cfg4_city")
    ap.add_argument("--codec", type=int, default=2, choices=[1, 2, 3], help="1 GTS, 2 GTS-Reuse, 3 Basic")
    ap.add_argument("--cull", action="store_true",
                    help="cone-culled compacted decode (FORMAT.md §7, extension f2) for a fixed view direction")
    ap.add_argument("--variable-widths", action="store_true",
                    help="per-meshlet attribute code widths (FORMAT.md VW, extension f1)")
    ap.add_argument("--index-format", default="u32", choices=["u32", "u8x4"],
                    help="u32: 3 global indices per triangle (default); u8x4: one local u8x4 word")
    ap.add_argument("--instances", type=int, default=1000, help="cfg4 instances per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-chunks", type=int, default=32, help="mc_decode_host pipeline depth (0/1 = serial)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and world == 1 and args.gpus > 1:
        log(f"--gpus {args.gpus} requested without torchrun; running 1 process")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
