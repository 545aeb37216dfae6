cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CFG=5 ROWS=${ROWS:-100000000} TAG=r02 bash scripts/gpu_prof_scan.sh
timeout 1200 python scripts/tile_trace.py --config 5 --n 100000000 > gpurun_out/tt_c5.txt 2>&1; tail -25 gpurun_out/tt_c5.txt
