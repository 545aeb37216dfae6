python scripts/prof_run.py --config 2 --reps 2 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_scan_tiles -s 1 -c 1 -o gpurun_out/prof_c2_scan_v7 python scripts/prof_run.py --config 2 --reps 2 > gpurun_out/ncu_c2.log 2>&1
python scripts/prof_run.py --config 5 --n 4000000 --reps 2 > gpurun_out/prof_plain5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_scan_tiles -s 1 -c 1 -o gpurun_out/prof_c5_scan_v7 python scripts/prof_run.py --config 5 --n 4000000 --reps 2 > gpurun_out/ncu_c5.log 2>&1
tail -n 2 gpurun_out/ncu_c2.log gpurun_out/ncu_c5.log
