python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -3
for cfg in 1 2; do
python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/q_$cfg.json 2>gpurun_out/q_$cfg.err
python -c "
import json; d=json.load(open('gpurun_out/q_$cfg.json')); s=d['config']['split_ms']
print('c$cfg', round(d['value']/1e6,1), 'Mq/s', {k: round(v,2) for k,v in s.items()}, 'exact/q', round(d['config']['per_query']['exact'],1), 'kd/q', round(d['config']['per_query']['kd_nodes'],1), 'frac', round(d['roofline']['frac'],2))"
done
