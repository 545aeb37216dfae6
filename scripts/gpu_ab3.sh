timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -1
VARIANTS="base||.ab/cur/x/y/cuda new||" CFGS="2 1" STEPS=10 bash scripts/gpu_ab.sh 2>&1
for v in base new; do P2M_LIB_DIR=/tmp/p2m_ab_$v python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v descend', round(d['config']['split_ms']['descend'],3), round(d['value']/1e6,1))"; done
