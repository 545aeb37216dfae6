"""Summarise one kernel of an .ncu-rep (ncu --set full): key metrics, stall mix, hottest CUDA lines.
usage: python scripts/ncu_summary2.py REP KERNEL_REGEX [TOP]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
run = lambda *a: subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", *a], capture_output=True, text=True).stdout
want = ['Duration', 'Elapsed Cycles', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'Executed Ipc Active', 'Issue Slots Busy', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Compute (SM) Throughput', 'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp',
        'Executed Instructions', 'Branch Efficiency', 'Grid Size', 'Block Limit Registers', 'Static Shared Memory Per Block']
r = csv.reader(io.StringIO(run('--page', 'details', '--csv'))); h = next(r)
seen = set()
for row in r:
    d = dict(zip(h, row))
    k = d.get('Metric Name')
    if k in want and k not in seen:
        seen.add(k)
        print(f"  {k:40s} {d['Metric Value']:>16s} {d.get('Metric Unit', '')}")
rr = list(csv.reader(io.StringIO(run('--page', 'raw', '--csv'))))
d = dict(zip(rr[0], rr[2]))
for k in ('gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
          'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
          'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
          'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
          'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum'):
    print(f"  {k:62s} {d.get(k)} {rr[1][rr[0].index(k)] if k in rr[0] else ''}")
print("  stall mix (warps stalled per issue):")
st = [(float(v), k) for k, v in d.items() if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('per_issue_active.ratio')]
for v, k in sorted(st, reverse=True)[:8]:
    print(f"    {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:24s} {v:.2f}")
rows = list(csv.reader(io.StringIO(run('--page', 'source', '--csv', '--print-source', 'sass,cuda'))))
cur = None; hdr = None; agg = []
for row in rows:
    if not row: continue
    if row[0] == 'File Path': cur = row[1].split('/')[-1]; continue
    if row[0] in ('Function Name',): continue
    if row[0] == 'Line No': hdr = row; continue
    if hdr and row[0].isdigit() and len(row) > 7:
        try: agg.append((int(row[4] or 0), cur, int(row[0]), row[1].strip()[:90], int(row[7] or 0)))
        except ValueError: pass
tot = sum(a[0] for a in agg) or 1
print(f"  hottest source lines by warp-stall samples ({tot} samples):")
for a in sorted(agg, reverse=True)[:top]:
    print(f"    {100 * a[0] / tot:5.1f}%  {a[1]}:{a[2]:<5d} inst {a[4] / 1e6:7.1f}M  {a[3]}")
toti = sum(a[4] for a in agg) or 1
print(f"  most executed source lines (warp instructions, {toti / 1e9:.1f} G attributed):")
for a in sorted(agg, key=lambda x: -x[4])[:top]:
    print(f"    {100 * a[4] / toti:5.1f}%  {a[1]}:{a[2]:<5d} inst {a[4] / 1e6:7.1f}M  stall {100 * a[0] / tot:4.1f}%  {a[3]}")
