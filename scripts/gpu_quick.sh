for ch in 4 6 8; do
P2M_E2E_CHUNKS=$ch python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/q_ch$ch.json 2>gpurun_out/q.err
python -c "
import json; d=json.load(open('gpurun_out/q_ch$ch.json'))
print('chunks $ch', round(d['value']/1e6,1), 'Mq/s e2e', round(d['e2e']['value']/1e6,1))"
done
