VARIANTS="e1|| e2|-DP2M_EARLY1=2|" CFGS="2 1 3 2" STEPS=10 bash scripts/gpu_ab.sh 2>&1
P2M_LIB_DIR=/tmp/p2m_ab_e2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_vs_oracle or stress or schedules" 2>&1 | tail -1
