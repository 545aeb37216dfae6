timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
VARIANTS="base||.ab/cur/x/y/cuda new||" CFGS="2 1 2 1" STEPS=10 bash scripts/gpu_ab.sh 2>&1
