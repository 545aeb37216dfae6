
for v in "" "P2M_E2E_CHUNKS=4" "P2M_E2E_CHUNKS=8" "P2M_E2E_CHUNKS=16"; do
  env $v P2M_E2E_TRACE=1 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/e2e.json 2>gpurun_out/e2e.err
  grep "e2e chunk" gpurun_out/e2e.err | tail -${TR:-0}
  python -c "
import json; d=json.load(open('gpurun_out/e2e.json')); print('[$v]', 'value', round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1), d['e2e']['rows_equal_device_path'])"
done
