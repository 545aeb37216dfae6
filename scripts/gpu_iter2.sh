# Iteration: fast GPU parity subset, then c5 / c2 / c1 device-resident benches (no CPU baseline).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
true
for c in ${CFGS:-5 2 1}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-pageable > gpurun_out/it_c$c.json 2> gpurun_out/it_c$c.err
  python - $c <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/it_c{c}.json").read().strip().splitlines()[-1])
    pq=d["config"]["per_query"]; sp=d["config"]["split_ms"]
    print(f"c{c}: {d['value']/1e6:.1f} Mq/s  e2e {d['e2e']['value']/1e6:.1f}  scan {sp['scan']:.2f} ms total {sp['total']:.2f}  exact {pq['exact']:.1f} passes {pq['filter_passes']:.1f} rare {pq['warp_rare_iters']:.1f} create {d['config']['create_s']} sbytes/row {d['roofline']['algorithmic_bytes_per_launch']/d['config']['queries_per_rank']:.0f}")
except Exception as e:
    print("c", c, "failed", e); print(open(f"gpurun_out/it_c{c}.err").read()[-2000:])
PY
done
