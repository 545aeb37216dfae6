# A/B of runtime knobs (environment variables) on ONE build, same box, same workloads.
# usage: VARIANTS="base|P2M_PROBE=0 probe|P2M_PROBE=1" CFGS="2 5" BIGN=20000000 bash scripts/gpu_env_ab.sh
set -u
mkdir -p gpurun_out
for cfg in ${CFGS}; do
  for v in ${VARIANTS}; do
    IFS="|" read -r name envs <<< "$v"
    envs=${envs//,/ }
    n=""
    if [ "$cfg" = 4 ] || [ "$cfg" = 5 ]; then n="--queries ${BIGN:-20000000}"; fi
    env $envs timeout 900 python bench.py --config $cfg $n --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/env_${name}_c$cfg.json 2> gpurun_out/env_${name}_c$cfg.err
    python -c "
import json; d=json.load(open('gpurun_out/env_${name}_c$cfg.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('$name c$cfg', round(d['value']/1e6,1), 'Mq/s scan', round(s['scan'],3), 'total', round(s['total'],3), 'E', round(pq['exact'],2), 'passes', round(pq.get('filter_passes',0),1), 'rare', round(pq.get('warp_rare_iters',0),1), 'e2e', round(d['e2e']['value']/1e6,1), 'rows_equal', d['e2e']['rows_equal_device_path'])" 2>&1 | tail -1
  done
done
