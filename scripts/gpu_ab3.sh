timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
declare -A V_ENV; V_ENV[twosort]="P2M_FUSED_FRONT=0"
VARIANTS="base||.ab/cur/x/y/cuda new|| twosort||" ENV_twosort="P2M_FUSED_FRONT=0" CFGS="2 1" STEPS=10 bash scripts/gpu_ab.sh 2>&1
for v in base new twosort; do
for n in 2500000 312500; do
env ${V_ENV[$v]:-} P2M_LIB_DIR=/tmp/p2m_ab_$v python bench.py --config 2 --queries $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/hv.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/hv.json')); s=d['config']['split_ms']; print('$v n $n', round(d['value']/1e6,1), {k: round(v,3) for k,v in s.items()}, 'e2e', round(d['e2e']['value']/1e6,1))"
done; done
