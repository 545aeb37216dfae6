for g in 0 1; do for cfg in 2 1; do
P2M_GATHER_Q=$g python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/hv.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/hv.json')); s=d['config']['split_ms']; print('gather $g c$cfg', round(d['value']/1e6,1), {k: round(v,3) for k,v in s.items()}, 'e2e', round(d['e2e']['value']/1e6,1), d['e2e']['rows_equal_device_path'])"
done; done
for g in 0 1; do
P2M_GATHER_Q=$g python bench.py --config 4 --queries 50000000 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/hv.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/hv.json')); s=d['config']['split_ms']; print('gather $g c4@50M', round(d['value']/1e6,1), {k: round(v,3) for k,v in s.items()})"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_vs_oracle or stress or schedules or geometric or concurrent" 2>&1 | tail -1
