python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/tr2.json 2> gpurun_out/tr2.err; echo rc=$?
tail -3 gpurun_out/tr2.err; cat gpurun_out/tr2.json | head -c 600; echo
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/tr2r.json 2> gpurun_out/tr2r.err; echo rc=$?
head -c 300 gpurun_out/tr2r.json; echo
