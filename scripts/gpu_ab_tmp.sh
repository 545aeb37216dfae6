for gd in 16 48 128 384; do for cfg in 2 1; do
P2M_GRID_DENSITY=$gd P2M_GRID_MAXRES=1024 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/hv.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/hv.json')); s=d['config']['split_ms']; pq=d['config']['per_query']; print('gd $gd c$cfg', round(d['value']/1e6,1), 'descend', round(s['descend'],3), 'cand', round(pq['kd_nodes'],1), 'scan', round(s['scan'],3), 'e2e', round(d['e2e']['value']/1e6,1))"
done; done
