#!/usr/bin/env python
"""Benchmark of the batched point-to-mesh query (BASELINE.json metric "point-to-mesh queries/sec
at 1/2/4/8 B200; % of HBM roofline").

A step = one pass of the hot path over one batch: Morton keys -> radix sort -> fused nearest-site
descent + pruned list scan, results scattered to input order, for one config batch per GPU (weak
scaling: every rank processes its own contiguous slice of the config's deterministic query
sequence on its own replica; no collective on the data path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Under torchrun (N>1) one process per GPU; the timed region is bracketed by a barrier +
torch.cuda.synchronize() on both sides, timed with CUDA events on the query stream, and the max
over ranks is reported by rank 0 as one JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "point-to-mesh queries/sec at 1/2/4/8 B200; % of HBM roofline"
CONFIG_N = {1: 1_000_000, 2: 10_000_000, 3: 20_000_000, 4: 100_000_000, 5: 100_000_000}
CONFIG_NAME = {
    1: "c1: icosphere L5 (10,242 V / 20,480 F), 1M uniform in AABBx1.2",
    2: "c2: noisy icosphere L5 (radial N(0,0.01)), 10M = 50% uniform AABBx1.2 + 50% surface+N(0,0.02)",
    3: "c3: capped cylinder 512x256 + cone 512, 20M uniform in AABBx1.3",
    4: "c4: jittered torus 1024x512 (1.05M F), 100M = 90% within 0.05 of surface + 10% AABBx1.5",
    5: "c5: 64-bump blob on icosphere L8 (1.31M F), 100M uniform in AABBx1.2",
}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock + throttle reasons sampled every 10 ms DURING the timed region (NVML in-process;
    nvidia-smi polling as a fallback)."""

    def __init__(self, gpu: int, period_s: float = 0.01):
        self.gpu = gpu
        self.period = period_s
        self.samples = []  # (sm_mhz, max_mhz, reason_bits)
        self._stop = threading.Event()
        self._t = None
        self.source = "nvml"

    def _run_nvml(self):
        import pynvml as N

        N.nvmlInit()
        try:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
            h = N.nvmlDeviceGetHandleByIndex(idx)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            get_r = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or N.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self._stop.is_set():
                self.samples.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), mx, int(get_r(h))))
                self._stop.wait(self.period)
        finally:
            N.nvmlShutdown()

    def _run_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={fields}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip().split(",")
                self.samples.append((float(out[0]), float(out[1]), int(out[2].strip(), 16)))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            self.source = "nvidia-smi"
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
        bits = 0
        for _, _, b in self.samples:
            bits |= b
        return {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(v for k, v in names.items() if bits & k), "samples": len(self.samples),
                "source": self.source}


def build_workload(cfg, rank, world, n_per_rank, build_threads, aux_corner_union):
    import paper_2605_00429_b200 as P

    t0 = time.perf_counter()
    V, F = P.mesh_config(cfg)
    t_mesh = time.perf_counter() - t0
    t0 = time.perf_counter()
    h = P.HostEngine.build(V, F, P.BuildConfig(n_threads=build_threads, aux_corner_union=aux_corner_union))
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    from paper_2605_00429_b200 import shard

    first, count = shard.rank_slice(rank, world, n_per_rank)
    q = P.gen_queries(cfg, V, F, first, count)
    t_q = time.perf_counter() - t0
    return V, F, h, q, {"mesh_s": round(t_mesh, 3), "build_s": round(t_build, 3), "queries_s": round(t_q, 3)}


def host_cores():
    """All host cores this process may use (torchrun exports OMP_NUM_THREADS=1; the CPU baseline
    deliberately ignores that and runs one OpenMP thread per core)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_oracle_rate(h, q, target_s=12.0, reference=True, threads=0):
    """Queries/s of the CPU query path on a bounded sample (prefix of the same workload)."""
    import oracle as O

    ref = reference and O.have_reference()
    oe = O.OracleEngine(h.arrays(), reference=ref)
    threads = threads or host_cores()
    n0 = min(len(q), 20000)
    t0 = time.perf_counter()
    oe.batch_query(q[:n0], prune=O.PRUNE_SAFE, threads=threads)
    dt0 = time.perf_counter() - t0
    n = int(min(len(q), max(n0, n0 * target_s / max(dt0, 1e-6))))
    t0 = time.perf_counter()
    oe.batch_query(q[:n], prune=O.PRUNE_SAFE, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "queries/s", "cores": threads, "kind": "reference" if ref else "port",
            "sample": f"first {n} queries of the workload ({dt:.1f} s, PRUNE_SAFE, OpenMP {threads} threads)"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU query path (oracle/_ref: REF geom.cpp + the restated
    query loop) on the host cores; rank 0 only."""
    if rank != 0:
        return
    import oracle as O

    cfg = args.config
    n_cfg = CONFIG_N[cfg]
    V, F, h, q, tb = build_workload(cfg, 0, 1, min(n_cfg, args.ref_sample), 0, (args.aux_table == "corner_union"))
    ref = O.have_reference()
    oe = O.OracleEngine(h.arrays(), reference=ref)
    threads = host_cores()
    n = len(q)
    for _ in range(args.warmup):
        oe.batch_query(q[: min(n, 20000)], threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oe.batch_query(q, prune=O.PRUNE_SAFE, threads=threads)
        times.append(time.perf_counter() - t0)
    t = max(1e-9, sum(times) / len(times))
    v = n / t
    line = {
        "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic config generator)",
        "impl": "reference",
        "config": {"workload": CONFIG_NAME[cfg], "queries_per_step": n, "build": tb,
                   "tables": args.aux_table},
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": threads,
                         "kind": "reference" if ref else "port",
                         "sample": f"{n} queries/step of the {CONFIG_NAME[cfg].split(':')[0]} workload"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--queries", type=int, default=0, help="override queries per rank")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=2_000_000)
    ap.add_argument("--aux-table", default="corner_union", choices=["corner_union", "ball"],
                    help="auxiliary-site tables: corner_union (default, REF/SPEC.md:413) or the literal single ball (406-414)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--scan-mode", type=int, default=0, help="0 grouped (default), 1 fused per-row")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2605_00429_b200 as P
    from paper_2605_00429_b200 import _lib as L
    from paper_2605_00429_b200 import shard

    if world > 1:
        # one rank per GPU over NCCL; the data path has no collective (barriers and the max-over-ranks
        # step time only).  If ranks must share a GPU (a smoke test on a 1-GPU box), NCCL refuses
        # duplicate devices, so the control plane falls back to gloo.
        ndev = torch.cuda.device_count()
        torch.cuda.set_device(local % ndev)
        if ndev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    cfg = args.config
    n = args.queries or CONFIG_N[cfg]
    ncpu = os.cpu_count() or 1
    V, F, h, q_host, tb = build_workload(cfg, rank, world, n, max(1, ncpu // world), (args.aux_table == "corner_union"))
    st = h.stats()
    eng = P.Engine(h, devices=[dev])
    lib = L.cuda()
    L.check(lib.p2m_set_scan_mode(eng.handle, args.scan_mode))

    stream = torch.cuda.current_stream()
    sptr = C.c_void_p(stream.cuda_stream)
    dq = torch.from_numpy(q_host).to(dev)
    ddist = torch.empty(n, dtype=torch.float64, device=dev)
    dcp = torch.empty((n, 3), dtype=torch.float64, device=dev)
    dface = torch.empty(n, dtype=torch.int32, device=dev)
    dsite = torch.empty(n, dtype=torch.int32, device=dev)
    dflags = torch.empty(n, dtype=torch.int32, device=dev)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    def step(counters=None):
        L.check(lib.p2m_query_device(eng.handle, 0, vp(dq), n, vp(ddist), vp(dcp), vp(dface), vp(dsite),
                                     vp(dflags), sptr, C.byref(counters) if counters is not None else None))

    # counters pass (untimed): algorithmic bytes per query
    cnt = L.Counters()
    step(cnt)
    torch.cuda.synchronize()
    c = cnt.as_dict()
    B_alg = 72 * n + 32 * c["kd_nodes_visited"] + 36 * c["candidates_visited"] + 72 * c["exact_evaluations"]

    for _ in range(args.warmup):
        step()
    kpq = C.c_int(0)
    L.check(lib.p2m_kernels_per_query(eng.handle, n, C.byref(kpq)))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    L.check(lib.p2m_set_profiling(eng.handle, 1))
    with ClockSampler(dev) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    split = (C.c_float * 6)()
    L.check(lib.p2m_last_timings(eng.handle, 0, split))
    L.check(lib.p2m_set_profiling(eng.handle, 0))
    split = [float(x) for x in split]
    ms_max = shard.max_over_ranks(ms, dist if world > 1 else None)
    value = n * world / (ms_max / 1e3)

    # e2e: the public host-buffer API (p2m_query) with pinned host memory, H2D + D2H inside
    qp = torch.from_numpy(q_host).pin_memory()
    o_dist = torch.empty(n, dtype=torch.float64).pin_memory()
    o_cp = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    o_face = torch.empty(n, dtype=torch.int32).pin_memory()
    o_site = torch.empty(n, dtype=torch.int32).pin_memory()
    o_flags = torch.empty(n, dtype=torch.int32).pin_memory()

    def e2e_call():
        L.check(lib.p2m_query(eng.handle, C.cast(C.c_void_p(qp.data_ptr()), L.dp), n,
                              C.cast(C.c_void_p(o_dist.data_ptr()), L.dp), C.cast(C.c_void_p(o_cp.data_ptr()), L.dp),
                              C.cast(C.c_void_p(o_face.data_ptr()), L.u32p), C.cast(C.c_void_p(o_site.data_ptr()), L.u32p),
                              C.cast(C.c_void_p(o_flags.data_ptr()), L.u32p), None))

    e2e_call()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_call()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    e2e_value = n * world / shard.max_over_ranks(e2e_s, dist if world > 1 else None)
    # the e2e rows must equal the device-resident rows (same engine, same inputs)
    same = bool(torch.equal(o_dist, ddist.cpu()) and torch.equal(o_face, dface.cpu()))
    if not same:
        print("WARNING: p2m_query rows differ from p2m_query_device rows on the same inputs "
              "(results must not depend on batching)", file=sys.stderr)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    # dominant kernel = the grouped list scan; its algorithmic bytes exclude the k-d descent
    # (that is the descend kernel's): 24 q + 40 out + 8 offsets + 36 C_q + 72 E_q per query
    B_scan = B_alg - 32 * c["kd_nodes_visited"]
    t_scan_s = split[4] / 1e3 if split[4] > 0 else ms / 1e3
    achieved = B_scan / t_scan_s / 1e9
    pipeline_gbs = B_alg / (split[5] / 1e3 if split[5] > 0 else ms / 1e3) / 1e9
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", f"traffic_c{cfg}.json")
    if os.path.exists(tr_path):
        try:
            with open(tr_path) as f:
                tr = json.load(f)
            traffic = tr.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_rate(h, q_host, target_s=12.0, reference=True)
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic config generator, fp64)",
        "config": {
            "workload": CONFIG_NAME[cfg], "queries_per_rank": n, "parallelism": f"queries sharded x{world}, structure replicated",
            "l2": "inputs larger than L2 (q 24 B + out 44 B per row; structure stays L2-resident by design)",
            "tables": {"corner_union": "aux corner-union (REF/SPEC.md:413)", "ball": "aux single ball (REF/SPEC.md:406-414)"}[args.aux_table],
            "build": tb, "n_sites": st["n_sites"], "n_faces": st["n_faces"], "list_avg": st["list_avg"],
            "list_max": st["list_max"],
            "per_query": {"candidates": c["candidates_visited"] / n, "exact": c["exact_evaluations"] / n,
                          "kd_nodes": c["kd_nodes_visited"] / n, "fallbacks": c["fallbacks"],
                          "filter_passes": c["filter_passes"] / n, "warp_rare_iters": c["warp_rare_iters"] / n},
            "split_ms": {"morton": split[0], "sort": split[1], "descend": split[2], "regroup_sort": split[3], "scan": split[4], "total": split[5]},
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "k_scan_tiles (site-tiled pruned list scan, exact fp64)",
                     # the DRAM bytes ncu measured for this kernel (traffic) over the live kernel time:
                     # the structure is L2/SMEM-resident, so real HBM use is a small fraction of peak
                     "measured_dram_gbs": (traffic / t_scan_s / 1e9) if traffic else None,
                     "measured_dram_frac": (traffic / t_scan_s / 1e9 / peak) if traffic else None,
                     "algorithmic_bytes_per_launch": B_scan,
                     "bytes_per_query": "72 + 36 C_q + 72 E_q (SURVEY.md 8(d) minus the 32 n_q of the descent kernel)",
                     "pipeline_algorithmic_gbs": pipeline_gbs, "pipeline_bytes_per_step": B_alg,
                     "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": 24 * n,
                "d2h_bytes_per_step": 44 * n, "api": "p2m_query (host pinned buffers, synchronous)",
                "rows_equal_device_path": same},
        "gpu_launches": int(kpq.value) * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
