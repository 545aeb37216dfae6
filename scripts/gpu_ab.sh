# A/B: build variant libraries on the box and bench each (same workload, same box).
# usage: VARIANTS="base|| minb2|-DP2M_SCAN_MINB=2| old||.ab/<commit>/x/y/cuda (git archive <commit> into .ab/, git-ignored)" CFGS="2 3" bash scripts/gpu_ab.sh
# entry = name|NVEXTRA|CUDADIR (CUDADIR empty = current sources); env ENV_<name> is exported for that variant
set -u
for v in ${VARIANTS}; do
  IFS="|" read -r name flags cdir <<< "$v"
  flags=${flags//,/ }
  dir=/tmp/p2m_ab_$name
  mkdir -p $dir
  extra=""
  [ -n "$cdir" ] && extra="CUDADIR=$cdir"
  make -s LIBDIR=$dir NVEXTRA="$flags" $extra $dir/libp2m_cuda.so > $dir/build.log 2>&1 || { echo "$name build failed"; tail -5 $dir/build.log; continue; }
  for cfg in ${CFGS}; do
    n=""
    if [ "$cfg" = 4 ] || [ "$cfg" = 5 ]; then n="--queries ${BIGN:-20000000}"; fi
    envv="ENV_$name"; envs="${!envv:-}"
    env $envs P2M_LIB_DIR=$dir timeout 900 python bench.py --config $cfg $n --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_${name}_c$cfg.json 2> gpurun_out/ab_${name}_c$cfg.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_${name}_c$cfg.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('$name c$cfg', round(d['value']/1e6,1), 'Mq/s scan', round(s['scan'],3), 'E', round(pq['exact'],2), 'passes', round(pq.get('filter_passes',0),1), 'e2e', round(d['e2e']['value']/1e6,1), 'rows_equal', d['e2e']['rows_equal_device_path'])" 2>&1 | tail -1
  done
done
