# final round check: the FULL GPU suite (incl. slow c3-c5 parity), smoke(), torchrun 2-rank functional run
set -u
O=gpurun_out/final; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_all.log 2>&1; tail -3 $O/pytest_gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 1 > $O/tr2.json 2> $O/tr2.err; echo rc=$?
head -c 400 $O/tr2.json; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $O/tr2r.json 2> $O/tr2r.err; echo rc=$?
head -c 300 $O/tr2r.json; echo
