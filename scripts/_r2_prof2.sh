cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_vs_oracle or fp32_prefilters or tiny or golden or vertex" > gpurun_out/it_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/it_tests.log
CFG=5 ROWS=100000000 TAG=r02 bash scripts/gpu_prof_scan.sh
