# ncu --set full (with source) of k_scan_tiles on c2 (10M rows) and on c5 (100M rows: one launch)
python scripts/prof_run.py --config 2 --reps 2 > gpurun_out/prof_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_scan_tiles -s 1 -c 1 -o gpurun_out/prof_c2_scan_${TAG:-v9} python scripts/prof_run.py --config 2 --reps 2 > gpurun_out/ncu_c2.log 2>&1
tail -n 1 gpurun_out/ncu_c2.log
