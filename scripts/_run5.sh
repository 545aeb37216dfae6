cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or stress or golden or table_miss or pageable" 2>&1 | tail -3
VARIANTS="compact|| union|-DP2M_COMPACT=0|" CFGS="2 5 1 4" BIGN=20000000 bash scripts/gpu_ab.sh
