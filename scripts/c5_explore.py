"""One build of a config, then three measurements on one GPU (JSON lines on stdout):
  sizes    device-resident p2m_query_device on prefixes of the batch (= the even strong-scaling
           shard of rank 0 at N = total/prefix GPUs; queries are iid, so every even shard is alike)
  spatial  the Morton-range strong-scaling shards (shard.spatial_shard's rule) of N = 2, 4, 8 ranks,
           each timed alone on this GPU -> the max over ranks is the N-GPU step time the data path
           would have (no collective on it; every GPU holds a full replica)
  e2e      p2m_query from pinned host buffers under several chunk schedules (an engine per schedule)
usage: python scripts/c5_explore.py CFG ROWS [sizes,spatial,e2e]"""
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L, shard

cfg, n = int(sys.argv[1]), int(sys.argv[2])
what = (sys.argv[3] if len(sys.argv) > 3 else "sizes,spatial,e2e").split(",")
V, F = P.mesh_config(cfg)
t0 = time.perf_counter()
h = P.HostEngine.build(V, F)
print(json.dumps({"build_s": round(time.perf_counter() - t0, 1)}), flush=True)
q = P.gen_queries(cfg, V, F, 0, n)
lib = L.cuda()
vp = lambda t: C.c_void_p(t.data_ptr())


def dev_time(eng, qh, reps=3):
    m = len(qh)
    dq = torch.from_numpy(np.ascontiguousarray(qh)).cuda()
    outs = [torch.empty(m, dtype=torch.float64, device="cuda"), torch.empty((m, 3), dtype=torch.float64, device="cuda")] + \
           [torch.empty(m, dtype=torch.int32, device="cuda") for _ in range(3)]
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    call = lambda: L.check(lib.p2m_query_device(eng.handle, 0, vp(dq), m, *[vp(t) for t in outs], sp, None))
    call(); call()
    torch.cuda.synchronize()
    L.check(lib.p2m_set_profiling(eng.handle, 1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        call()
    e1.record(s)
    torch.cuda.synchronize()
    split = (C.c_float * 6)()
    L.check(lib.p2m_last_timings(eng.handle, 0, split))
    L.check(lib.p2m_set_profiling(eng.handle, 0))
    return e0.elapsed_time(e1) / reps, [round(float(x), 3) for x in split]


if "sizes" in what or "spatial" in what:
    eng = P.Engine(h)
    t_full, sp_full = dev_time(eng, q)
    print(json.dumps({"sizes": n, "ms": round(t_full, 3), "Mqps": round(n / t_full / 1e3, 1), "split": sp_full}), flush=True)
if "sizes" in what:
    for div in (2, 4, 8, 16, 32):
        m = n // div
        t, sp = dev_time(eng, q[:m])
        print(json.dumps({"sizes": m, "even_ranks": div, "ms": round(t, 3), "Mqps": round(m / t / 1e3, 1),
                          "speedup_vs_1": round(t_full / t, 2), "split": sp}), flush=True)
if "spatial" in what:
    a = h.arrays()
    box = shard.morton_box(a["site_xyz"][a["site_kind"] != 1])
    keys = np.concatenate([shard.morton_keys(q[i:i + (1 << 23)], box).astype(np.int64) for i in range(0, n, 1 << 23)])
    counts = np.bincount(keys, minlength=1 << 21)
    for world, ppr in ((2, 1), (4, 1), (8, 1), (2, 4), (4, 4), (8, 4), (8, 8), (8, 16)):
        bnd = shard.spatial_bounds(counts, world * ppr)
        part = (np.searchsorted(bnd, keys, side="right") - 1) % world
        ts, ms_ = [], []
        for r in range(world):
            sel = np.flatnonzero(part == r)
            t, _ = dev_time(eng, q[sel], reps=2)
            ts.append(round(t, 2)); ms_.append(int(len(sel)))
        print(json.dumps({"spatial_ranks": world, "parts_per_rank": ppr, "rows": ms_, "ms": ts, "max_ms": max(ts),
                          "speedup_vs_1": round(t_full / max(ts), 2)}), flush=True)
    del keys
if "sizes" in what or "spatial" in what:
    del eng
    torch.cuda.empty_cache()
if "e2e" in what:
    qp = torch.from_numpy(q).pin_memory()
    outs = [torch.empty(n, dtype=torch.float64).pin_memory(), torch.empty((n, 3), dtype=torch.float64).pin_memory()] + \
           [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(3)]
    dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), L.dp)
    up = lambda t: C.cast(C.c_void_p(t.data_ptr()), L.u32p)
    scheds = os.environ.get("SCHEDS", "default;chunks=1;chunks=2;chunks=3;chunks=4;0.4,1,0.4,0.2;0.5,1,0.5,0;0.25,1.5,0.5,0;0.125,2,0.5,0;0.3,1,0.35,0.05").split(";")
    ref = None
    for sc in scheds:
        os.environ.pop("P2M_E2E_SCHED", None); os.environ.pop("P2M_E2E_CHUNKS", None)
        if sc.startswith("chunks="):
            os.environ["P2M_E2E_CHUNKS"] = sc.split("=")[1]
        elif sc != "default":
            os.environ["P2M_E2E_SCHED"] = sc
        eng = P.Engine(h)
        call = lambda: L.check(lib.p2m_query(eng.handle, dp(qp), n, dp(outs[0]), dp(outs[1]), up(outs[2]), up(outs[3]), up(outs[4]), None))
        call()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter(); call(); ts.append(time.perf_counter() - t0)
        t = min(ts)
        d = outs[0].numpy().tobytes()
        same = ref is None or d == ref
        ref = ref or d
        print(json.dumps({"e2e_sched": sc, "Mqps": round(n / t / 1e6, 1), "ms": round(t * 1e3, 1), "rows_equal": same}), flush=True)
        del eng
        torch.cuda.empty_cache()
