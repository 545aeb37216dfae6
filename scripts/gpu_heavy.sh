for thr in 1024 256 64 16; do
  for n in 10000000 2500000 312500; do
    P2M_HEAVY_E=$thr python bench.py --config 2 --queries $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/hv.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/hv.json')); s=d['config']['split_ms']; print('thr $thr n $n', round(d['value']/1e6,1), 'scan', round(s['scan'],3), 'e2e', round(d['e2e']['value']/1e6,1))"
  done
done
