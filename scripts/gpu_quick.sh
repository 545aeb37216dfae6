python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" 2>&1 | grep -E "passed|failed|Error" | tail -4
for tab in corner_union ball; do for cfg in 1 2; do
python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --aux-table $tab > gpurun_out/q_${cfg}_$tab.json 2>gpurun_out/q_$cfg.err
python -c "
import json; d=json.load(open('gpurun_out/q_${cfg}_$tab.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('c$cfg $tab', round(d['value']/1e6,1), 'Mq/s', {k: round(v,2) for k,v in s.items()}, 'C/q', round(pq['candidates'],1), 'E/q', round(pq['exact'],1), 'frac', round(d['roofline']['frac'],2))"
done; done
