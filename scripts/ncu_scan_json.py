"""Roofline evidence of the scan phase from one ncu --set full capture (scripts/gpu_prof_scan.sh):
DRAM bytes, duration and pipe utilisation of k_scan_tiles + k_scan_small (the two kernels of one
scan phase; ncu serialises them) -> profiles/<round>/ncu_scan_c<cfg>.json, tagged with the sha256
of the CUDA sources that were profiled.  bench.py uses the file only when its own sources have the
same hash and the row count matches (same build, same workload).

usage: python scripts/ncu_scan_json.py REP CFG ROWS OUT.json [LIB]"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # src_sha256: the hash bench.py matches the evidence against

rep, cfg, rows, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
lib = sys.argv[5] if len(sys.argv) > 5 else os.path.join(os.path.dirname(__file__), "..", "paper_2605_00429_b200", "lib", "libp2m_cuda.so")
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(txt)))
hdr = rr[0]
kern = []
for row in rr[2:]:
    d = dict(zip(hdr, row))
    name = d.get("Kernel Name", "")
    if "k_scan_tiles" in name or "k_scan_small" in name or "k_scan_warpq" in name:
        kern.append(d)
if not kern:
    sys.exit("no scan kernels in " + rep)


def f(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


# one launch of each kernel (the last capture of each name)
last = {}
for d in kern:
    last["tiles" if "k_scan_tiles" in d["Kernel Name"] else "small"] = d
ks = list(last.values())
unit = {h: rr[1][i] for i, h in enumerate(hdr)}
tscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}[unit.get("gpu__time_duration.sum", "nsecond")]
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12}


def b(d, k):
    return f(d, k) * bscale.get(unit.get(k, "byte"), 1)


try:
    PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    PEAK = 6650.0
t = [f(d, "gpu__time_duration.sum") * tscale for d in ks]
T = sum(x for x in t if x == x)


def w(k):
    # duration-weighted over the kernels that report the metric (a launch with no work has none)
    num = den = 0.0
    for d, ti in zip(ks, t):
        v = f(d, k)
        if v == v and ti == ti:
            num += v * ti
            den += ti
    return num / den if den else float("nan")


def nz(x):
    return x if x == x else 0.0


dram = sum(nz(b(d, "dram__bytes_read.sum")) + nz(b(d, "dram__bytes_write.sum")) for d in ks)
res = {
    "config": cfg, "rows": rows, "kernels": [d["Kernel Name"][:60] for d in ks],
    "lib_sha256": hashlib.sha256(open(lib, "rb").read()).hexdigest(),
    "src_sha256": bench.src_sha256(),
    "gpu_time_s": T, "dram_bytes_per_launch": dram, "dram_gbs_under_ncu": dram / T / 1e9,
    "dram_pct": 100.0 * dram / T / 1e9 / PEAK,
    "l2_hit_pct": w("lts__t_sector_hit_rate.pct"),
    "fp64_pipe_pct": w("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "fma_pipe_pct": w("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_pct": w("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "lsu_pct": w("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "issue_slots_pct": w("sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
    "ipc": w("sm__inst_executed.avg.per_cycle_active"),
    "source": os.path.basename(rep),
}
top = max(("dram", res["dram_pct"]), ("fp64 pipe", res["fp64_pipe_pct"]), ("fma pipe", res["fma_pipe_pct"]),
          ("issue slots", res["issue_slots_pct"]), key=lambda x: x[1] if x[1] == x[1] else -1)
res["binding"] = f"{top[0]} ({top[1]:.0f}% of peak): the scan is instruction-issue / latency bound, not HBM-bound"
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
with open(out, "w") as fp:
    json.dump(res, fp, indent=1)
print(json.dumps(res))
