cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or fp32_prefilters or tiny or golden or vertex" > gpurun_out/it_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/it_tests.log
export ENV_curw="P2M_SCAN_WARP=1"
VARIANTS="cur|| curw|| head||.ab/head/paper_2605_00429_b200/csrc/cuda" CFGS="5 2 1" BIGN=100000000 STEPS=3 bash scripts/gpu_ab.sh
