cd $GRAFT_REPO_ROOT
VARIANTS="lb6|P2M_X=0" CFGS="2 5 4 1 3" BIGN=20000000 bash scripts/gpu_env_ab.sh
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or large_configs or stress or golden or schedules" 2>&1 | tail -5
