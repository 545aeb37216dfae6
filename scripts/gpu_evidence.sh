# Evidence pass for the current HEAD: GPU tests, default bench, reference arm, launch list of the
# same bench command, ncu --set full of the dominant kernels.  Usage: TAG=r01b bash scripts/gpu_evidence.sh
set -u
TAG=${TAG:-r01b}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > $O/gpu.txt
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
fi
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err; tail -c 600 $O/bench_default.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch.log 2>&1
timeout 600 python scripts/prof_run.py --config 2 --reps 2 > $O/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_scan_tiles|k_descend" -s 2 -c 2 \
    -o $O/prof_c2 python scripts/prof_run.py --config 2 --reps 2 > $O/ncu_full.log 2>&1
tail -n 2 $O/ncu_launch.log $O/ncu_full.log
for cfg in 1 ${CFGS:-}; do
  st=10; [ "$cfg" -ge 3 ] && st=3
  timeout 1500 python bench.py --config $cfg --steps $st --warmup 3 --e2e-steps 2 > $O/bench_c$cfg.json 2> $O/bench_c$cfg.err
  tail -c 300 $O/bench_c$cfg.json
done
