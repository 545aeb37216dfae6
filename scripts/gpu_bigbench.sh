for cfg in 3 4 5; do
  python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/big_c$cfg.json 2> gpurun_out/big_c$cfg.err
  echo "c$cfg rc=$?"; grep -E "Maximum resident|Elapsed" gpurun_out/big_c$cfg.err
  python -c "
import json; d=json.load(open('gpurun_out/big_c$cfg.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('c$cfg', round(d['value']/1e6,1), 'Mq/s', {k: round(v,2) for k,v in s.items()}, 'C/q', round(pq['candidates'],1), 'E/q', round(pq['exact'],1), 'e2e', round(d['e2e']['value']/1e6,1), 'cpu', d['cpu_baseline'], 'build', d['config']['build'])" 2>&1 | tail -2
done
