# c2 throughput vs batch size (device-resident and host-buffer paths)
for n in 312500 1000000 2500000 10000000 40000000; do
  python bench.py --config 2 --queries $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/sz.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sz.json')); s=d['config']['split_ms']; print($n, round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), round(s['total'],3))"
done
