O=gpurun_out/r01f; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "schedules or concurrent" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for cfg in 4 5; do
  timeout 1500 python bench.py --config $cfg --steps 3 --warmup 3 --e2e-steps 2 > $O/bench_c$cfg.json 2> $O/bench_c$cfg.err
  tail -c 200 $O/bench_c$cfg.json
done
