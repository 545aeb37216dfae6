cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or fp32_prefilters or tiny or golden or vertex" > gpurun_out/it_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/it_tests.log
export ENV_t32="P2M_HEAVY_E=0 P2M_LONG_TILE=32" ENV_t64="P2M_HEAVY_E=0 P2M_LONG_TILE=64"
VARIANTS="tight|| prev||.ab/prev/paper_2605_00429_b200/csrc/cuda t32|| t64||" CFGS="5 2" BIGN=100000000 STEPS=3 bash scripts/gpu_ab.sh
