# one iteration: GPU tests (non-slow), then c1/c2 quick bench and c3..c5 at reduced steps
set -u
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -4
bash scripts/gpu_quick.sh
for cfg in ${BIG_CFGS:-3 4 5}; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/it_c$cfg.json 2> gpurun_out/it_c$cfg.err
  python -c "
import json; d=json.load(open('gpurun_out/it_c$cfg.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('c$cfg', round(d['value']/1e6,1), 'Mq/s', {k: round(v,2) for k,v in s.items()}, {k: round(v,1) for k, v in pq.items()}, 'e2e', round(d['e2e']['value']/1e6,1))" 2>&1 | tail -1
done
