VARIANTS="base|| nr|-DP2M_VISIT_RETEST=0| s32|-DP2M_DK_SQRT32=1| both|-DP2M_VISIT_RETEST=0,-DP2M_DK_SQRT32=1|" CFGS="2 1 3" STEPS=10 bash scripts/gpu_ab.sh 2>&1
P2M_LIB_DIR=/tmp/p2m_ab_both timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_vs_oracle or stress" 2>&1 | tail -1
