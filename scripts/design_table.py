"""The DESIGN.md section 7 results table from a directory of bench lines (bench_default.json = c5,
bench_c1..c4.json).  usage: python scripts/design_table.py profiles/r02/final"""
import json, os, sys
d = sys.argv[1]
rows = []
for cfg, name in ((5, "bench_default.json"), (4, "bench_c4.json"), (3, "bench_c3.json"), (2, "bench_c2.json"), (1, "bench_c1.json")):
    p = os.path.join(d, name)
    if not os.path.exists(p):
        continue
    try:
        x = json.loads(open(p).read().strip().split("\n")[-1])
    except Exception:
        continue
    c = x["config"]
    n = c["queries_total"]
    cpu = x["cpu_baseline"]["value"] if x.get("cpu_baseline") else None
    par = x.get("parity") or {}
    g = lambda v: f"{v / 1e9:.3f} G q/s" if v >= 1e8 else f"{v / 1e6:.1f} M q/s"
    rows.append(f"| c{cfg}, {n // 1000000} M{' (bench default)' if cfg == 5 else ''} | **{g(x['value'])}** ({x['ms_per_step']:.1f} ms) | "
                f"{g(x['e2e']['value'])} | {g(x['e2e_pageable']['value']) if x.get('e2e_pageable') else '—'} | "
                f"{g(cpu) if cpu else '—'} | {x['e2e']['value'] / cpu:.0f}× | {c['per_query']['candidates']:.0f} | {c['per_query']['exact']:.1f} | "
                f"{x['roofline']['frac']:.3f} | {par.get('bit_exact', '—')}/{par.get('rows', '—')} |")
print("| Config | GPU device-resident | GPU e2e (pinned host) | GPU e2e (pageable) | CPU reference (16 cores) | speed-up e2e | C/q | E/q | roofline frac | parity rows (bit-exact/checked) |")
print("|---|---|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
