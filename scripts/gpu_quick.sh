for cfg in 1 2; do
python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/q_${cfg}.json 2>gpurun_out/q.err
python -c "
import json; d=json.load(open('gpurun_out/q_${cfg}.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('c$cfg', round(d['value']/1e6,1), 'Mq/s', {k: round(v,2) for k,v in s.items()}, {k: round(v,1) for k, v in pq.items()}, 'e2e', round(d['e2e']['value']/1e6,1))"
done
