cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "device_image or device_built_grid or table_miss or pageable" 2>&1 | grep -E "descent ms|passed|failed|Error|assert" | head
VARIANTS="sdk|| base||.ab/base/paper_2605_00429_b200/csrc/cuda" CFGS="5 2 1" BIGN=20000000 bash scripts/gpu_ab.sh
CFG=5 ROWS=20000000 TAG=r02 bash scripts/gpu_prof_scan.sh
