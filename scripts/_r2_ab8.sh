cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/it_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/it_tests.log
export ENV_cmpw="P2M_SCAN_WARP=1"
VARIANTS="cmp|| nocmp|-DP2M_COMPACT=0| cmpw||" CFGS="5 2 1" BIGN=100000000 STEPS=3 bash scripts/gpu_ab.sh
