"""Debug: per-tile durations of k_scan_tiles (P2M_TILE_TRACE) for one device-path call."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ctypes as C
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=312500)
a = ap.parse_args()
V, F = P.mesh_config(a.config)
h = P.HostEngine.build(V, F)
q = P.gen_queries(a.config, V, F, 0, a.n)
eng = P.Engine(h)
dq = torch.from_numpy(q).cuda()
outs = [torch.empty(a.n, dtype=torch.float64, device="cuda"), torch.empty((a.n, 3), dtype=torch.float64, device="cuda")] + \
       [torch.empty(a.n, dtype=torch.int32, device="cuda") for _ in range(3)]
vp = lambda t: C.c_void_p(t.data_ptr())
for it in range(3):
    path = f"/tmp/tt_{it}.bin"
    os.environ["P2M_TILE_TRACE"] = path
    L.check(L.cuda().p2m_query_device(eng.handle, 0, vp(dq), a.n, *[vp(t) for t in outs], None, None))
    torch.cuda.synchronize()
del os.environ["P2M_TILE_TRACE"]
t = np.fromfile(path, dtype=np.uint64).reshape(-1, 4)
t = t[t[:, 1] > 0]
cyc = (t[:, 3] >> 8).astype(np.float64)
ms = cyc / 1.965e6
print(f"config {a.config} n {a.n}: tiles {len(t)}  sum {ms.sum():.1f} CTA-ms  mean {ms.mean()*1e3:.1f} us  p50 {np.median(ms)*1e3:.1f} us  max {ms.max()*1e3:.1f} us")
o = np.argsort(-ms)[:15]
for i in o:
    print(f"  site {int(t[i,0]):6d} rows {int(t[i,1]):4d} list {int(t[i,2]):6d}  {ms[i]*1e3:8.1f} us")
rows = t[:, 1]
for lo, hi in [(1, 8), (8, 32), (32, 64), (64, 128), (128, 256), (256, 257)]:
    m = (rows >= lo) & (rows < hi)
    print(f"  rows [{lo},{hi}): tiles {m.sum():6d}  CTA-ms {ms[m].sum():8.1f}  mean {ms[m].mean()*1e3 if m.any() else 0:7.1f} us")
L_ = t[:, 2]
for lo, hi in [(0, 256), (256, 1024), (1024, 4096), (4096, 16384), (16384, 65536), (65536, 1 << 40)]:
    m = (L_ >= lo) & (L_ < hi)
    print(f"  list [{lo},{hi}): tiles {m.sum():6d}  rows {int(rows[m].sum()):9d}  CTA-ms {ms[m].sum():8.1f}  max {ms[m].max() if m.any() else 0:7.2f} ms")
srt = np.sort(ms)[::-1]
for fr in (0.001, 0.01, 0.1):
    k = max(1, int(len(srt) * fr))
    print(f"  top {fr*100:.1f}% tiles: {srt[:k].sum():8.1f} CTA-ms of {ms.sum():.1f}")
print(f"  ideal wall at 592 CTA slots: {ms.sum()/592:.1f} ms")
