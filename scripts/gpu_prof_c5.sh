# new-feature GPU tests, then one ncu --set full capture of k_scan_tiles on c5 (20M rows)
timeout 1500 python -m pytest tests/test_tables.py tests/test_walk.py -m "gpu and not slow" -x -q 2>&1 | tail -4
python scripts/prof_run.py --config 5 --n 20000000 --reps 2 > gpurun_out/prof_plain5.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_scan_tiles -s 1 -c 1 -o gpurun_out/prof_c5_scan_v8 python scripts/prof_run.py --config 5 --n 20000000 --reps 2 > gpurun_out/ncu_c5.log 2>&1
tail -n 2 gpurun_out/ncu_c5.log
