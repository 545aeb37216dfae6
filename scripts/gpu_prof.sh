python scripts/prof_run.py --config 2 --reps 2 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_scan_tiles -s 1 -c 1 -o gpurun_out/prof_c2_scan_v4 python scripts/prof_run.py --config 2 --reps 2 > gpurun_out/ncu_c2.log 2>&1
python scripts/prof_run.py --config 1 --reps 2 > gpurun_out/prof_plain1.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_descend -s 1 -c 1 -o gpurun_out/prof_c1_descend python scripts/prof_run.py --config 1 --reps 2 > gpurun_out/ncu_c1d.log 2>&1
tail -n 3 gpurun_out/ncu_c2.log gpurun_out/ncu_c1d.log
