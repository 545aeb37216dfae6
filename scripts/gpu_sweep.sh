python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for cfg in 1 2; do for LT in 32 64; do for HE in 256 1024 4096; do
P2M_HEAVY_E=$HE P2M_LONG_TILE=$LT python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw_${cfg}_${LT}_${HE}.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/sw_${cfg}_${LT}_${HE}.json')); s=d['config']['split_ms']
print('c${cfg} LT=${LT} HE=${HE}', round(d['value']/1e6,1), 'Mq/s scan', round(s['scan'],2), 'desc', round(s['descend'],2), 'exact/q', round(d['config']['per_query']['exact'],1))"
done; done; done
