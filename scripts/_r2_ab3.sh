cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or fp32_prefilters or tiny or golden or vertex" > gpurun_out/it_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/it_tests.log
P2M_SCAN_WARP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or fp32_prefilters or tiny or golden or vertex" > gpurun_out/it_tests_w.log 2>&1; echo "warp tests exit $?"; tail -2 gpurun_out/it_tests_w.log
export ENV_warp="P2M_SCAN_WARP=1" ENV_warplpt="P2M_SCAN_WARP=1 P2M_TILE_ORDER=1" ENV_warpm3="P2M_SCAN_WARP=1"
VARIANTS="base|| warp|| warplpt|| warpm3|-DP2M_SMALL_MINB=3|" CFGS="5 2 1" BIGN=100000000 STEPS=3 bash scripts/gpu_ab.sh
