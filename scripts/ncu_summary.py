"""Summarise an .ncu-rep: key metrics + hottest SASS lines (used to write profiles/*.md)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
want = ['Duration','Elapsed Cycles','Achieved Occupancy','Theoretical Occupancy','Registers Per Thread','Executed Ipc Active',
        'Issue Slots Busy','Memory Throughput','DRAM Throughput','L1/TEX Hit Rate','L2 Hit Rate','Compute (SM) Throughput',
        'Warp Cycles Per Issued Instruction','Avg. Active Threads Per Warp','Executed Instructions','Branch Efficiency',
        'Grid Size','Block Limit Registers','Block Limit Shared Mem','Dynamic Shared Memory Per Block','Static Shared Memory Per Block']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out)); h = next(r)
name = None
for row in r:
    d = dict(zip(h, row))
    name = d.get('Kernel Name', name)
    if d.get('Metric Name') in want:
        print(f"  {d['Metric Name']:40s} {d['Metric Value']:>16s} {d.get('Metric Unit','')}")
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
for k, v in zip(rr[0], rr[2]):
    if k in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__cycles_active.avg', 'sm__cycles_active.max',
             'lts__t_sector_hit_rate.pct', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
             'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
             'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum'):
        print(f"  {k:60s} {v}")
if len(sys.argv) > 2:
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]; data = rows[2:]
    iA, iS, iE, iW = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[iE] or 0) for r in data)
    top = sorted(data, key=lambda r: -int(r[iW] or 0))[:int(sys.argv[2])]
    print(f"  total warp instructions {tot:,}; top stall-sampled SASS:")
    for r in sorted(top, key=lambda r: int(r[iA], 16)):
        print(f"    {r[iA][-5:]} {int(r[iE] or 0)/1e6:8.1f}M  stall {r[iW]:>7}  {r[iS][:80]}")
