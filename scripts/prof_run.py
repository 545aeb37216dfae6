"""Minimal driver for ncu: build config C, run p2m_query_device `reps` times on device buffers."""
import argparse, ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--aux-ball", action="store_true")
a = ap.parse_args()
N = {1: 1_000_000, 2: 10_000_000, 3: 20_000_000, 4: 100_000_000, 5: 100_000_000}
n = a.n or N[a.config]
V, F = P.mesh_config(a.config)
h = P.HostEngine.build(V, F, P.BuildConfig(aux_corner_union=not a.aux_ball))
q = P.gen_queries(a.config, V, F, 0, n)
eng = P.Engine(h)
lib = L.cuda()
L.check(lib.p2m_set_scan_mode(eng.handle, a.mode))
dq = torch.from_numpy(q).cuda()
outs = [torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda")] + \
       [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(3)]
vp = lambda t: C.c_void_p(t.data_ptr())
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(a.reps):
    L.check(lib.p2m_query_device(eng.handle, 0, vp(dq), n, *[vp(t) for t in outs], s, None))
torch.cuda.synchronize()
print("ok", n)
