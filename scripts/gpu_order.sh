timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
for v in "P2M_TILE_ORDER=0" "P2M_TILE_ORDER=1" "P2M_TILE_ORDER=2"; do
for n in 312500 2500000 10000000; do
  env $v python bench.py --config 2 --queries $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/sz.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sz.json')); s=d['config']['split_ms']; print('[$v]', $n, round(d['value']/1e6,1), 'scan', round(s['scan'],3), 'e2e', round(d['e2e']['value']/1e6,1), d['e2e']['rows_equal_device_path'])"
done
for cfg in 3 5; do
  env $v python bench.py --config $cfg --queries 20000000 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sz.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sz.json')); s=d['config']['split_ms']; print('[$v]', 'c$cfg 20M', round(d['value']/1e6,1), 'scan', round(s['scan'],3), d['e2e']['rows_equal_device_path'])"
done
done
