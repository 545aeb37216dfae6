cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
P2M_WARP_MIN_CHUNKS=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or fp32_prefilters or tiny or golden or vertex" > gpurun_out/it_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/it_tests.log
export ENV_h2="P2M_WARP_MIN_CHUNKS=2" ENV_h4="P2M_WARP_MIN_CHUNKS=4" ENV_h8="P2M_WARP_MIN_CHUNKS=8" ENV_h1="P2M_WARP_MIN_CHUNKS=1"
VARIANTS="base|| h1|| h2|| h4|| h8||" CFGS="5 2 1" BIGN=100000000 STEPS=3 bash scripts/gpu_ab.sh
