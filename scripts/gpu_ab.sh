# A/B: build variant libraries on the box (same sources, different NVEXTRA) and bench each.
# usage: VARIANTS="base:  minb2:-DP2M_SCAN_MINB=2" CFGS="2 5" bash scripts/gpu_ab.sh
set -u
for v in ${VARIANTS}; do
  name=${v%%:*}; flags=${v#*:}
  dir=/tmp/p2m_ab_$name
  mkdir -p $dir
  make -s LIBDIR=$dir NVEXTRA="$flags" $dir/libp2m_cuda.so > $dir/build.log 2>&1 || { echo "$name build failed"; tail -5 $dir/build.log; continue; }
  for cfg in ${CFGS}; do
    n=""
    [ "$cfg" = 4 ] || [ "$cfg" = 5 ] && n="--queries ${BIGN:-20000000}"
    P2M_LIB_DIR=$dir timeout 900 python bench.py --config $cfg $n --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_${name}_c$cfg.json 2> gpurun_out/ab_${name}_c$cfg.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_${name}_c$cfg.json')); s=d['config']['split_ms']; pq=d['config']['per_query']
print('$name c$cfg', round(d['value']/1e6,1), 'Mq/s scan', round(s['scan'],2), 'E', round(pq['exact'],1), 'passes', round(pq['filter_passes'],1))" 2>&1 | tail -1
  done
done
