timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ico3" 2>&1 | grep -v "^$" | tail -30
P2M_E2E_TRACE=1 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 >/dev/null | grep "e2e chunk" | tail -8
P2M_E2E_TRACE=1 P2M_E2E_CHUNKS=4 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 >/dev/null | grep "e2e chunk" | tail -4
