# round-1 evidence: plain bench (default args), launch list of the same command, full capture of k_scan_tiles
set -x
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
python scripts/prof_run.py --config 2 --reps 2 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_scan_tiles -s 1 -c 1 -o gpurun_out/prof_c2_scan_r01 \
    python scripts/prof_run.py --config 2 --reps 2 > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/ncu_launch.log gpurun_out/ncu_full.log
