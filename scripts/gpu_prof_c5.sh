# one ncu --set full capture of k_scan_tiles on c5 (20 M rows), after a plain run of the same command
mkdir -p gpurun_out/c5prof
timeout 1200 python scripts/prof_run.py --config 5 --n 20000000 --reps 1 > gpurun_out/c5prof/plain.log 2>&1 && \
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:"k_scan_tiles|k_scan_small" -c 2 \
    -o gpurun_out/c5prof/prof_c5 python scripts/prof_run.py --config 5 --n 20000000 --reps 1 > gpurun_out/c5prof/ncu.log 2>&1
tail -n 2 gpurun_out/c5prof/plain.log gpurun_out/c5prof/ncu.log
