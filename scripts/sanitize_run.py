"""Small end-to-end run of every device path, for compute-sanitizer."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L
V, F = P.mesh_config(2)
h = P.HostEngine.build(V, F)
q = np.concatenate([P.gen_queries(2, V, F, 0, 30000), np.random.default_rng(0).uniform(-30, 30, (200, 3)), V[:50]])
for devs in ([0], [0, 0]):
    e = P.Engine(h, devices=devs)
    for mode in (0, 1):
        L.check(L.cuda().p2m_set_scan_mode(e.handle, mode))
        r = e.batch_query(q)
    e.batch_query(np.zeros((0, 3)))
    e.batch_query(q[:1])
V1, F1 = P.icosphere(1)
h1 = P.HostEngine.build(V1, F1)
P.Engine(h1).batch_query(np.random.default_rng(1).uniform(-2, 2, (5000, 3)))
print("sanitize run ok", r.counters)
