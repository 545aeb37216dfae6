for sc in 1 2; do
P2M_SMALL_CHUNKS=$sc python bench.py --config 5 --queries 20000000 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/hv.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/hv.json')); s=d['config']['split_ms']; print('c5 sc $sc', round(d['value']/1e6,1), 'scan', round(s['scan'],3), 'e2e', round(d['e2e']['value']/1e6,1))"
done
