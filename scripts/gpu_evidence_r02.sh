# Round-2 evidence pass for HEAD: default bench (c5), reference arm, scan-phase ncu (--set full +
# launch list of the bench command), then the full -m gpu suite.  TAG=r02a bash scripts/gpu_evidence_r02.sh
set -u
cd ${GRAFT_REPO_ROOT:-.}
TAG=${TAG:-r02a}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > $O/gpu.txt
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err; echo "bench exit $?"; tail -c 400 $O/bench_default.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref exit $?"
CFG=5 ROWS=100000000 TAG=$TAG bash scripts/gpu_prof_scan.sh
cp -r gpurun_out/prof_c5 $O/ 2>/dev/null
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "tests exit $?"; tail -3 $O/pytest_gpu.log
fi
