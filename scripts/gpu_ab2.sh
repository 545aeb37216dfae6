timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
VARIANTS="new|| head||scripts/ab_old/x/y/cuda" CFGS="2 3 5" BIGN=20000000 STEPS=5 bash scripts/gpu_ab.sh
for v in new head; do
  for n in 2500000; do
    P2M_LIB_DIR=/tmp/p2m_ab_$v python bench.py --config 2 --queries $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sz.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/sz.json')); s=d['config']['split_ms']; print('$v', $n, round(d['value']/1e6,1), 'scan', round(s['scan'],3))"
  done
done
