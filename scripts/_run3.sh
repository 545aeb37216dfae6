cd $GRAFT_REPO_ROOT
VARIANTS="lb2s|P2M_X=0" CFGS="2 5 1" BIGN=20000000 bash scripts/gpu_env_ab.sh
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pageable or table_miss or parity_vs_oracle or stress or golden or chunk_schedules" 2>&1 | tail -5
python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/bench_c2_new.json 2> gpurun_out/bench_c2_new.err; tail -c 3000 gpurun_out/bench_c2_new.json; tail -5 gpurun_out/bench_c2_new.err
