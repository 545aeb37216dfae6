"""A/B of engine-creation environment knobs on one build of a config: one engine per variant, the
device-resident step time (CUDA events, split by phase) and the per-query counters of each.
usage: python scripts/env_ab.py CFG ROWS "default;P2M_NO_DEEP_SEED=1;A=1,B=2" [reps]"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L

cfg, n = int(sys.argv[1]), int(sys.argv[2])
variants = sys.argv[3].split(";")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
V, F = P.mesh_config(cfg)
h = P.HostEngine.build(V, F)
q = P.gen_queries(cfg, V, F, 0, n)
lib = L.cuda()
dq = torch.from_numpy(q).cuda()
outs = [torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda")] + \
       [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(3)]
vp = lambda t: C.c_void_p(t.data_ptr())
s = torch.cuda.current_stream()
sp = C.c_void_p(s.cuda_stream)
ref = None
touched = set()
for var in variants:
    for k in touched:
        os.environ.pop(k, None)
    if var != "default":
        for kv in var.split(","):
            k, v = kv.split("=")
            os.environ[k] = v
            touched.add(k)
    eng = P.Engine(h)
    call = lambda cnt=None: L.check(lib.p2m_query_device(eng.handle, 0, vp(dq), n, *[vp(t) for t in outs], sp,
                                                          C.byref(cnt) if cnt is not None else None))
    cnt = L.Counters()
    call(cnt)
    torch.cuda.synchronize()
    c = cnt.as_dict()
    call()
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
    ms = e0.elapsed_time(e1) / reps
    d = outs[0].cpu().numpy().tobytes() + outs[2].cpu().numpy().tobytes()
    same = ref is None or d == ref
    ref = ref or d
    print(json.dumps({"cfg": cfg, "rows": n, "variant": var, "ms": round(ms, 3), "Mqps": round(n / ms / 1e3, 1),
                      "scan_ms": round(float(split[4]), 3), "rows_equal_first": same,
                      "exact_q": round(c["exact_evaluations"] / n, 2), "passes_q": round(c["filter_passes"] / n, 2),
                      "rare_iters_q": round(c["warp_rare_iters"] / n, 2),
                      "struct_B_q": round(c["structure_bytes"] / n, 1)}), flush=True)
    del eng
    torch.cuda.empty_cache()
