# Round-2 final evidence pass for the current build.  TAG=final bash scripts/gpu_final_r02.sh
#  1 scan-phase ncu (--set full) + launch list of the bench command -> profiles-ready JSON/text
#  2 default bench (c5) with that same-build evidence in place, reference arm
#  3 benches of c1..c4, 4 full -m gpu suite, smoke(), 5 a 2-rank torchrun run (spatial split default)
set -u
cd ${GRAFT_REPO_ROOT:-.}
TAG=${TAG:-final}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > $O/gpu.txt
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
CFG=5 ROWS=100000000 TAG=$TAG bash scripts/gpu_prof_scan.sh
mkdir -p profiles/r02/$TAG
cp gpurun_out/prof_c5/ncu_scan_c5.json gpurun_out/prof_c5/scan_tiles_c5.txt gpurun_out/prof_c5/scan_warp_c5.txt gpurun_out/prof_c5/launches_c5.csv profiles/r02/$TAG/ 2>/dev/null
cp gpurun_out/prof_c5/ncu_scan_c5.json gpurun_out/prof_c5/scan_tiles_c5.txt gpurun_out/prof_c5/scan_warp_c5.txt gpurun_out/prof_c5/launches_c5.csv $O/ 2>/dev/null
rm -f gpurun_out/prof_c5/scan_c5.ncu-rep
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench exit $?"; tail -c 600 $O/bench_default.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref exit $?"
for cfg in 1 2 4 3; do
  timeout 1500 python bench.py --config $cfg --steps 5 --warmup 3 > $O/bench_c$cfg.json 2> $O/bench_c$cfg.err; echo "c$cfg exit $?"
  python -c "
import json; d=json.load(open('$O/bench_c$cfg.json')); print('c$cfg', round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1), 'pageable', round(d['e2e_pageable']['value']/1e6,1), 'cpu', round(d['cpu_baseline']['value']/1e6,2), 'parity', d['parity'])"
done
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "tests exit $?"; tail -3 $O/pytest_gpu.log
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $O/smoke.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config 2 --steps 3 --warmup 3 > $O/bench_2rank_c2.json 2> $O/bench_2rank_c2.err; echo "2-rank exit $?"; tail -c 400 $O/bench_2rank_c2.json
