timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
for sd in 0 3 6 8; do
for cfg in 2 1; do
P2M_SEEDS=$sd python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/hv.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/hv.json')); s=d['config']['split_ms']; pq=d['config']['per_query']; print('seeds $sd c$cfg', round(d['value']/1e6,1), 'scan', round(s['scan'],3), 'E', round(pq['exact'],2), 'passes', round(pq['filter_passes'],1), 'visits', round(pq['warp_rare_iters'],1), 'e2e', round(d['e2e']['value']/1e6,1))"
done; done
