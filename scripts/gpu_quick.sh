set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -15
for m in 0 1; do python bench.py --steps 5 --warmup 3 --scan-mode $m --no-cpu-baseline > gpurun_out/bench_m$m.json 2> gpurun_out/bench_m$m.err; echo rc=$?; tail -3 gpurun_out/bench_m$m.err; done
python bench.py --steps 5 --warmup 3 --config 1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
cat gpurun_out/bench_m0.json gpurun_out/bench_c1.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['value']/1e6, 'Mq/s', d['config']['split_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value']/1e6)"
