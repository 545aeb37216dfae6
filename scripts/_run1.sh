cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
VARIANTS="base|P2M_PROBE=0 probe|P2M_PROBE=1" CFGS="2 5 4 1" BIGN=20000000 bash scripts/gpu_env_ab.sh
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or large_configs or stress or golden" 2>&1 | tail -5
