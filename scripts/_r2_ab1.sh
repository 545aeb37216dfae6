cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or fp32_prefilters or tiny or golden or vertex or schedules" > gpurun_out/it_tests.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/it_tests.log
VARIANTS="base|| minb3|-DP2M_SCAN_MINB=3|" CFGS="5 2 1" BIGN=100000000 STEPS=3 bash scripts/gpu_ab.sh
