cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -x -q > gpurun_out/it_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/it_tests.log; grep -E "FAILED|Error" gpurun_out/it_tests.log | head -5
CFGS="5 2 1" bash scripts/gpu_iter2.sh 2>&1 | tail -4
