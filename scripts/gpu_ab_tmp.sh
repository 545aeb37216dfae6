VARIANTS="base||.ab/cur/x/y/cuda early||" CFGS="2 1 3 2" STEPS=10 bash scripts/gpu_ab.sh 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_vs_oracle or stress or schedules" 2>&1 | tail -1
