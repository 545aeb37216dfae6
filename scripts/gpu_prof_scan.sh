# Roofline evidence for bench.py: ncu --set full of one scan phase (k_scan_tiles + k_scan_small) on
# config CFG at the bench's row count, after a plain run of the same command; summary JSON (with the
# library hash) + text summaries under gpurun_out/prof_c$CFG/.
# usage: CFG=5 ROWS=100000000 TAG=r02 bash scripts/gpu_prof_scan.sh
set -u
CFG=${CFG:-5}; ROWS=${ROWS:-100000000}; TAG=${TAG:-r02}
d=gpurun_out/prof_c$CFG; mkdir -p $d
timeout 1200 python scripts/prof_run.py --config $CFG --n $ROWS --reps 1 > $d/plain.log 2>&1 || { echo "plain run failed"; tail -5 $d/plain.log; exit 1; }
timeout 2400 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"k_scan_(tiles|small|warpq)" -c 2 -o $d/scan_c$CFG -f \
    python scripts/prof_run.py --config $CFG --n $ROWS --reps 1 > $d/ncu.log 2>&1 || { echo "ncu failed"; tail -5 $d/ncu.log; }
python scripts/ncu_scan_json.py $d/scan_c$CFG.ncu-rep $CFG $ROWS $d/ncu_scan_c$CFG.json
python scripts/ncu_summary2.py $d/scan_c$CFG.ncu-rep "k_scan_tiles" 30 > $d/scan_tiles_c$CFG.txt 2>&1
python scripts/ncu_summary2.py $d/scan_c$CFG.ncu-rep "k_scan_(small|warpq)" 40 > $d/scan_warp_c$CFG.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $d/launches_c$CFG.csv \
    python bench.py --config $CFG --queries $ROWS --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-pageable > $d/launches.log 2>&1
tail -3 $d/launches.log
