for nb in 0 1; do
if [ $nb = 1 ]; then export P2M_NO_BATCH=1; else unset P2M_NO_BATCH; fi
for cfg in 2 5; do
python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --queries 10000000 > gpurun_out/q_${cfg}.json 2>gpurun_out/q.err
python -c "
import json; d=json.load(open('gpurun_out/q_${cfg}.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('c$cfg nobatch=$nb', round(d['value']/1e6,1), 'Mq/s', 'scan', round(s['scan'],2), 'E/q', round(pq['exact'],1))"
done; done
