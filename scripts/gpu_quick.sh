python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" 2>&1 | grep -E "passed|failed|Error|assert" | tail -6
for seed in 0 1; do for cfg in 1 2; do
if [ $seed = 1 ]; then export P2M_NO_SEED=1; else unset P2M_NO_SEED; fi
python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/q_${cfg}.json 2>gpurun_out/q.err
python -c "
import json; d=json.load(open('gpurun_out/q_${cfg}.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('c$cfg noseed=$seed', round(d['value']/1e6,1), 'Mq/s', {k: round(v,2) for k,v in s.items()}, 'E/q', round(pq['exact'],1), 'e2e', round(d['e2e']['value']/1e6,1))"
done; done
