for hd in 0 500 1500 4000; do
for c in "1 0" "2 0" "2 2500000" "2 625000"; do set -- $c
P2M_HEAVY_DIV=$hd python bench.py --config $1 --queries $2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/hv.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/hv.json')); s=d['config']['split_ms']; print('hd $hd c$1 n $2', round(d['value']/1e6,1), 'scan', round(s['scan'],3), 'e2e', round(d['e2e']['value']/1e6,1))"
done; done
