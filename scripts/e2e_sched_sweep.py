"""Host-buffer (p2m_query) schedule sweep on one config: one build, one batch, an engine per schedule
(P2M_E2E_SCHED = first,growth,cap,tail as fractions of the batch, read at engine creation).
usage: python scripts/e2e_sched_sweep.py CFG ROWS "sched1;sched2;..." """
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L

cfg, n = int(sys.argv[1]), int(sys.argv[2])
scheds = sys.argv[3].split(";")
V, F = P.mesh_config(cfg)
h = P.HostEngine.build(V, F)
q = P.gen_queries(cfg, V, F, 0, n)
qp = torch.from_numpy(q).pin_memory()
outs = [torch.empty(n, dtype=torch.float64).pin_memory(), torch.empty((n, 3), dtype=torch.float64).pin_memory()] + \
       [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(3)]
dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), L.dp)
up = lambda t: C.cast(C.c_void_p(t.data_ptr()), L.u32p)
ref = None
for sc in scheds:
    if sc == "default":
        os.environ.pop("P2M_E2E_SCHED", None)
    else:
        os.environ["P2M_E2E_SCHED"] = sc
    eng = P.Engine(h)
    call = lambda: L.check(L.cuda().p2m_query(eng.handle, dp(qp), n, dp(outs[0]), dp(outs[1]), up(outs[2]), up(outs[3]), up(outs[4]), None))
    call()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); call(); ts.append(time.perf_counter() - t0)
    t = min(ts)
    d = outs[0].numpy().copy()
    same = ref is None or d.tobytes() == ref
    ref = ref or d.tobytes()
    print(f"sched {sc:24s} {n / t / 1e6:8.1f} M q/s  ({t * 1e3:.1f} ms)  rows_equal {same}", flush=True)
    del eng
