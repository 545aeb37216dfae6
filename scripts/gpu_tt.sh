cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python scripts/tile_trace.py --config ${CFG:-5} --n ${ROWS:-100000000} > gpurun_out/tt_c${CFG:-5}.txt 2>&1; tail -40 gpurun_out/tt_c${CFG:-5}.txt
