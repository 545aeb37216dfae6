#!/usr/bin/env python
"""Benchmark of the batched point-to-mesh query (BASELINE.json metric "point-to-mesh queries/sec
at 1/2/4/8 B200; % of HBM roofline").

Default workload: config c5 (BASELINE.json configs[4]: 64-bump blob on an icosphere L8, 1.31 M
faces, 100 M queries uniform in AABBx1.2) -- the 100M-query config the metric is quoted on at
1/2/4/8 GPUs, and it fits one GPU.  A step = one pass of the hot path over the batch on each GPU:
Morton keys -> radix sort -> nearest-site descent -> regroup by site -> pruned list scan, results
in input order (p2m_query_device on device-resident queries).

Multi-GPU (torchrun, one process per GPU): STRONG scaling by default -- the one 100 M batch is
sharded over the ranks (Morton-range partitions by default, so every GPU keeps the rows per site
of the single-GPU run; --split even: contiguous slices); rank 0 builds
the engine once and the other ranks load its EngineIndexFile.  No collective on the data path
(barriers and the max-over-ranks step time only).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
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
# bytes per row moved by the scan kernels besides the structure: q (24) + row index (4) in,
# distance (8) + closest point (24) + face id (4) out
ROW_BYTES = 64


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


def host_cores():
    """All host cores this process may use (torchrun exports OMP_NUM_THREADS=1; the CPU baseline
    deliberately ignores that and runs one OpenMP thread per core)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def build_engine(cfg, rank, world, build_threads, aux_corner_union, index_dir=None, barrier=None,
                 table_device=None):
    """The host engine of config cfg.  With several ranks, rank 0 builds it once and saves the
    EngineIndexFile (REF/SPEC.md:588-591); the other ranks load it (mesh re-validated, hash checked)."""
    import paper_2605_00429_b200 as P

    t0 = time.perf_counter()
    V, F = P.mesh_config(cfg)
    t_mesh = time.perf_counter() - t0
    info = {"mesh_s": round(t_mesh, 3)}
    cfgb = P.BuildConfig(n_threads=build_threads, aux_corner_union=aux_corner_union)
    path = None
    if world > 1 and index_dir:
        os.makedirs(index_dir, exist_ok=True)
        path = os.path.join(index_dir, f"c{cfg}_{int(aux_corner_union)}_{os.getpid() if rank == 0 else 0}.p2mx")
    if world > 1 and index_dir:
        t0 = time.perf_counter()
        if rank == 0:
            h = P.HostEngine.build(V, F, cfgb, table_device=table_device)
            info["build_s"] = round(time.perf_counter() - t0, 3)
            h.save(path)
            names = [path]
        else:
            names = [None]
        import torch.distributed as dist

        dist.broadcast_object_list(names, src=0)
        if rank != 0:
            t0 = time.perf_counter()
            h = P.HostEngine.load(names[0], V, F)
            info["load_s"] = round(time.perf_counter() - t0, 3)
        if barrier:
            barrier()
        if rank == 0:
            try:
                os.remove(path)
            except OSError:
                pass
    else:
        t0 = time.perf_counter()
        h = P.HostEngine.build(V, F, cfgb, table_device=table_device)
        info["build_s"] = round(time.perf_counter() - t0, 3)
    st = h.stats()
    info["build_split_s"] = {"voronoi": round(st["t_voronoi_s"], 3), "augment": round(st["t_augment_s"], 3),
                             "tables": round(st["t_tables_s"], 3), "total": round(st["t_total_s"], 3)}
    info["tables_on"] = "host" if table_device is None else f"cuda:{table_device}"
    return V, F, h, info


def rank_queries(cfg, V, F, rank, world, n_total, scaling, split, key_box, parts_per_rank=1):
    """This rank's rows of the batch: strong scaling shards ONE batch of n_total rows (even slices or
    Morton-range partitions), weak scaling gives every rank its own n_total rows."""
    import paper_2605_00429_b200 as P
    from paper_2605_00429_b200 import shard

    t0 = time.perf_counter()
    if scaling == "weak":
        first, count = shard.rank_slice(rank, world, n_total)
        q = P.gen_queries(cfg, V, F, first, count)
        desc = f"rows [{first}, {first + count}) of the config's query sequence"
    elif split == "even" or world == 1:
        first, count = shard.device_shard(n_total, world, rank)
        q = P.gen_queries(cfg, V, F, first, count)
        desc = f"even slice [{first}, {first + count}) of the {n_total}-row batch"
    else:
        gen = lambda a, b: P.gen_queries(cfg, V, F, a, b)  # noqa: E731
        q, idx = shard.spatial_shard(gen, n_total, world, rank, key_box, parts_per_rank=parts_per_rank)
        desc = (f"Morton-range part {rank}/{world} ({parts_per_rank} interleaved ranges) of the "
                f"{n_total}-row batch ({len(q)} rows)")
    return q, {"queries_s": round(time.perf_counter() - t0, 3), "rows": desc}


def cpu_reference_rows(h, q, target_s=12.0, threads=0):
    """The reference CPU query path (oracle/_ref when built: REF geom.cpp + the restated loop) on a
    bounded prefix of the same workload: its rate and its rows (for the in-line parity check)."""
    import oracle as O

    ref = O.have_reference()
    oe = O.OracleEngine(h.arrays(), reference=ref)
    threads = threads or host_cores()
    n0 = min(len(q), 20000)
    t0 = time.perf_counter()
    oe.batch_query(q[:n0], prune=O.PRUNE_SAFE, threads=threads)
    dt0 = time.perf_counter() - t0
    n = int(min(len(q), max(n0, n0 * target_s / max(dt0, 1e-6))))
    t0 = time.perf_counter()
    rows = oe.batch_query(q[:n], prune=O.PRUNE_SAFE, threads=threads)
    dt = time.perf_counter() - t0
    info = {"value": n / dt, "unit": "queries/s", "cores": threads, "kind": "reference" if ref else "port",
            "sample": f"first {n} queries of the workload ({dt:.1f} s, PRUNE_SAFE, OpenMP {threads} threads)"}
    return info, rows, n


def parity_rows(ref, gpu, n):
    """Rows bit-identical between the reference CPU path and the GPU (distance, closest point, face,
    site, flags -- every field, compared as bits)."""
    ok = np.ones(n, bool)
    ok &= ref["distance"][:n].view(np.uint64) == gpu["distance"][:n].view(np.uint64)
    ok &= (ref["closest"][:n].reshape(n, 3).view(np.uint64) == gpu["closest"][:n].reshape(n, 3).view(np.uint64)).all(1)
    for k in ("face", "site", "flags"):
        ok &= ref[k][:n].astype(np.uint32) == gpu[k][:n].astype(np.uint32)
    return int(ok.sum())


def src_sha256():
    """Hash of the CUDA sources, the ABI header and the build flags: identifies the build the ncu
    evidence was taken on (a hash of the .so itself changes with every relink)."""
    import glob

    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2605_00429_b200", "csrc", "cuda", "*.cu*")))
    files += [os.path.join(ROOT, "include", "p2m.h"), os.path.join(ROOT, "Makefile")]
    for p in files:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def ncu_evidence(cfg, rows, sha):
    """DRAM traffic and pipe utilisation of the scan kernels from an ncu --set full capture of THIS
    build (profiles/*/ncu_scan_c{cfg}.json, written by scripts/ncu_scan_json.py, carries the
    sha256 of the CUDA sources it profiled): used only if the hash and the row count match."""
    import glob

    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "**", f"ncu_scan_c{cfg}.json"), recursive=True), reverse=True):
        try:
            with open(p) as f:
                d = json.load(f)
        except Exception:
            continue
        if d.get("src_sha256") == sha and int(d.get("rows", -1)) == int(rows):
            d["file"] = os.path.relpath(p, ROOT)
            return d
    return None


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU query path (oracle/_ref: REF geom.cpp + the restated
    query loop) on all host cores, on a bounded sample of the same workload; rank 0 only."""
    if rank != 0:
        return
    import oracle as O
    import paper_2605_00429_b200 as P

    cfg = args.config
    n_cfg = args.queries or CONFIG_N[cfg]
    V, F, h, tb = build_engine(cfg, 0, 1, 0, args.aux_table == "corner_union")
    ref = O.have_reference()
    oe = O.OracleEngine(h.arrays(), reference=ref)
    threads = host_cores()
    # size one step to ~args.ref_step_s of CPU work (calibrated on a 20k-row prefix)
    qc = P.gen_queries(cfg, V, F, 0, min(n_cfg, 20000))
    t0 = time.perf_counter()
    oe.batch_query(qc, prune=O.PRUNE_SAFE, threads=threads)
    rate0 = len(qc) / max(time.perf_counter() - t0, 1e-6)
    n = int(min(n_cfg, max(len(qc), rate0 * args.ref_step_s)))
    q = P.gen_queries(cfg, V, F, 0, n)
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
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.scaling == "strong" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic config generator)",
        "impl": "reference",
        "config": {"workload": CONFIG_NAME[cfg], "queries_per_step": n, "build": tb,
                   "tables": args.aux_table},
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": threads,
                         "kind": "reference" if ref else "port",
                         "sample": f"first {n} queries/step of the {CONFIG_NAME[cfg].split(':')[0]} workload"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--queries", type=int, default=0, help="override the batch size (rows)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default): N GPUs share one batch; weak: every GPU gets a full batch")
    ap.add_argument("--split", default="auto", choices=["auto", "even", "spatial"],
                    help="strong scaling: even contiguous slices or Morton-range (spatial) partitions; "
                         "auto = spatial for N > 1 (rows per site stay those of the 1-GPU run)")
    ap.add_argument("--parts-per-rank", type=int, default=8,
                    help="spatial split: Morton ranges per rank, dealt round-robin (load balance)")
    ap.add_argument("--index-dir", default=os.environ.get("P2M_INDEX_DIR", "/tmp/p2m_bench_index"),
                    help="N>1: where rank 0 writes the EngineIndexFile the other ranks load")
    ap.add_argument("--table-device", type=int, default=-1,
                    help="run the builder's table phase on this GPU (bit-identical tables); -1 = host")
    ap.add_argument("--ref-step-s", type=float, default=6.0, help="--impl reference: CPU seconds per step")
    ap.add_argument("--aux-table", default="corner_union", choices=["corner_union", "ball"],
                    help="auxiliary-site tables: corner_union (default, REF/SPEC.md:413) or the literal single ball (406-414)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-s", type=float, default=12.0, help="CPU seconds of the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-pageable", action="store_true")
    ap.add_argument("--scan-mode", type=int, default=0, help="0 grouped (default), 1 fused per-row")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.split == "auto":
        args.split = "spatial" if env_int("WORLD_SIZE", 1) > 1 and args.scaling == "strong" else "even"

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
    barrier = (lambda: dist.barrier()) if world > 1 else None
    dev = torch.cuda.current_device()
    cfg = args.config
    n_total = args.queries or CONFIG_N[cfg]
    ncpu = host_cores()
    tdev = dev if args.table_device >= 0 else None
    V, F, h, tb = build_engine(cfg, rank, world, max(1, ncpu // world) if world > 1 and not args.index_dir else ncpu,
                               args.aux_table == "corner_union", args.index_dir, barrier, tdev)
    st = h.stats()
    t0 = time.perf_counter()
    eng = P.Engine(h, devices=[dev])
    torch.cuda.synchronize()
    create_s = time.perf_counter() - t0
    lib = L.cuda()
    L.check(lib.p2m_set_scan_mode(eng.handle, args.scan_mode))
    arrays = h.arrays()
    key_box = shard.morton_box(arrays["site_xyz"][arrays["site_kind"] != 1])
    q_host, tq = rank_queries(cfg, V, F, rank, world, n_total, args.scaling, args.split, key_box,
                              args.parts_per_rank)
    tb.update(tq)
    n = len(q_host)

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

    # counters pass (untimed): per-query counts and the scan's structure bytes (the roofline's bytes)
    cnt = L.Counters()
    step(cnt)
    torch.cuda.synchronize()
    c = cnt.as_dict()

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
    rows_job = n_total if args.scaling == "strong" else n_total * world
    value = rows_job / (ms_max / 1e3)
    gpu_rows = {"distance": ddist.cpu().numpy(), "closest": dcp.cpu().numpy(), "face": dface.cpu().numpy(),
                "site": dsite.cpu().numpy(), "flags": dflags.cpu().numpy()}

    # e2e: the public host-buffer API (p2m_query), H2D + D2H inside the timed region, from pinned
    # host memory (the contract's e2e) and from ordinary pageable numpy arrays (the numpy caller)
    qp = torch.from_numpy(q_host).pin_memory()
    o_dist = torch.empty(n, dtype=torch.float64).pin_memory()
    o_cp = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    o_face = torch.empty(n, dtype=torch.int32).pin_memory()
    o_site = torch.empty(n, dtype=torch.int32).pin_memory()
    o_flags = torch.empty(n, dtype=torch.int32).pin_memory()
    dpp = lambda t: C.cast(C.c_void_p(t.data_ptr()), L.dp)  # noqa: E731
    upp = lambda t: C.cast(C.c_void_p(t.data_ptr()), L.u32p)  # noqa: E731

    def e2e_call():
        L.check(lib.p2m_query(eng.handle, dpp(qp), n, dpp(o_dist), dpp(o_cp), upp(o_face), upp(o_site),
                              upp(o_flags), None))

    def timed(fn, k):
        fn()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            fn()
        return (time.perf_counter() - t0) / k

    e2e_s = timed(e2e_call, args.e2e_steps)
    e2e_value = rows_job / shard.max_over_ranks(e2e_s, dist if world > 1 else None)
    # the e2e rows must equal the device-resident rows (same engine, same inputs)
    same = bool(np.array_equal(o_dist.numpy().view(np.uint64), gpu_rows["distance"].view(np.uint64))
                and np.array_equal(o_face.numpy(), gpu_rows["face"]))
    if not same:
        print("WARNING: p2m_query rows differ from p2m_query_device rows on the same inputs "
              "(results must not depend on batching)", file=sys.stderr)
    del qp, o_dist, o_cp, o_face, o_site, o_flags
    pageable = None
    if not args.no_pageable:
        qn = np.ascontiguousarray(q_host)
        pd = np.empty(n); pc = np.empty((n, 3)); pf = np.empty(n, np.uint32); ps = np.empty(n, np.uint32)
        pfl = np.empty(n, np.uint32)

        def e2e_pageable():
            L.check(lib.p2m_query(eng.handle, L.ptr(qn), n, L.ptr(pd), L.ptr(pc), L.ptr(pf, L.u32p),
                                  L.ptr(ps, L.u32p), L.ptr(pfl, L.u32p), None))

        pg_s = timed(e2e_pageable, max(1, args.e2e_steps - 1))
        pageable = {"value": rows_job / shard.max_over_ranks(pg_s, dist if world > 1 else None),
                    "unit": "queries/s", "api": "p2m_query (pageable numpy buffers)",
                    "rows_equal_device_path": bool(np.array_equal(pd.view(np.uint64), gpu_rows["distance"].view(np.uint64)))}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    # Roofline of the dominant kernel (the scan phase: k_scan_warpq || k_scan_tiles).  Algorithmic
    # bytes per launch = 64 B per row (q + row index in, distance + closest point + face out) + the
    # structure bytes the scan kernels load, counted by the kernels themselves in the counters pass:
    # each staged batch (face ids + face disks) once per tile or warp tile, group records once per
    # visit, each face record once per exact test -- never per row.  Over the scan's mean time
    # measured with CUDA events on the query stream in the timed region.
    t_scan_s = split[4] / 1e3 if split[4] > 0 else ms / 1e3
    B_scan = ROW_BYTES * n + c["structure_bytes"]
    achieved = B_scan / t_scan_s / 1e9
    sha = src_sha256()
    ev = ncu_evidence(cfg, n, sha)
    traffic = ev["dram_bytes_per_launch"] if ev else None
    compute = None
    if ev:
        compute = {"fp64_pipe_pct": ev.get("fp64_pipe_pct"), "fma_pipe_pct": ev.get("fma_pipe_pct"),
                   "issue_slots_pct": ev.get("issue_slots_pct"), "dram_pct": ev.get("dram_pct"),
                   "binding": ev.get("binding"), "source": ev["file"]}
    cpu = None
    parity = None
    if world == 1 and not args.no_cpu_baseline:
        cpu, ref_rows, n_s = cpu_reference_rows(h, q_host, target_s=args.cpu_s)
        parity = {"rows": n_s, "bit_exact": parity_rows(ref_rows, gpu_rows, n_s),
                  "checker": "oracle/_ref (REF geom.cpp + the restated query loop)" if cpu["kind"] == "reference"
                  else "oracle (C restatement)",
                  "fields": "distance, closest point, face, site, flags (bitwise)"}
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic config generator, fp64)",
        "config": {
            "workload": CONFIG_NAME[cfg], "queries_total": rows_job, "queries_per_rank": n,
            "parallelism": f"queries sharded x{world} ({args.split if args.scaling == 'strong' else 'weak'}), structure replicated",
            "l2": "inputs larger than L2 (q 24 B + out 44 B per row); the read-only structure is not flushed",
            "tables": {"corner_union": "aux corner-union (REF/SPEC.md:413)", "ball": "aux single ball (REF/SPEC.md:406-414)"}[args.aux_table],
            "build": tb, "create_s": round(create_s, 3), "n_sites": st["n_sites"], "n_faces": st["n_faces"],
            "list_avg": st["list_avg"], "list_max": st["list_max"],
            "per_query": {"candidates": c["candidates_visited"] / n, "exact": c["exact_evaluations"] / n,
                          "kd_nodes": c["kd_nodes_visited"] / n, "fallbacks": c["fallbacks"],
                          "filter_passes": c["filter_passes"] / n, "warp_rare_iters": c["warp_rare_iters"] / n},
            "scan_tiles": c["scan_tiles"],
            "split_ms": {"morton": split[0], "sort": split[1], "descend": split[2], "regroup_sort": split[3], "scan": split[4], "total": split[5]},
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "scan phase: k_scan_warpq || k_scan_tiles (site-tiled pruned list scan, exact fp64)",
                     "algorithmic_bytes_per_launch": B_scan,
                     "bytes_model": "64 B/row (q, row index, distance, closest point, face) + the structure bytes the "
                                    "scan kernels load, counted in-kernel: per tile the list's chunk points and "
                                    "cylinders (16 + 32 B per chunk) and 76 B of offsets/meta; per visited chunk its "
                                    "batch cylinders (32 B each); per staged batch 36 B/entry (face id + face disk); "
                                    "96 B face record per exact evaluation (per queued pair on the warp-tile path, per warp "
                                    "visit on the CTA path)",
                     "measured_dram_gbs": (traffic / t_scan_s / 1e9) if traffic else None,
                     "compute": compute,
                     "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": 24 * n,
                "d2h_bytes_per_step": 44 * n, "api": "p2m_query (host pinned buffers, synchronous)",
                "rows_equal_device_path": same},
        "e2e_pageable": pageable,
        "parity": parity,
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
