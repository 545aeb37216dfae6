import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_00429_b200 as P, oracle as O
V, F = P.icosphere(3); h = P.HostEngine.build(V, F)
q = np.random.default_rng(3).uniform(-1.3, 1.3, size=(20000, 3))
r = P.Engine(h).batch_query(q)
ref = O.OracleEngine(h.arrays()).batch_query(q)
bad = np.flatnonzero(r.face != ref["face"])
print("bad", len(bad))
d = r.distance[bad] - ref["distance"][bad]
print("dist diff: >0", (d > 0).sum(), "==0", (d == 0).sum(), "<0", (d < 0).sum(), "max", d.max())
print("gpu faces", r.face[bad[:8]], "ref", ref["face"][bad[:8]])
print("exact/q gpu", r.counters["exact_evaluations"] / len(q), "ref", ref["counters"]["exact_evaluations"] / len(q))
