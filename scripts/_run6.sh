cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "device_image or table_miss or pageable or brute_force and 2" 2>&1 | tail -3
CFG=5 ROWS=20000000 TAG=r02 bash scripts/gpu_prof_scan.sh
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 4000 gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
