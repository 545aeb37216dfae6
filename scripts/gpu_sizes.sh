for n in 312500 1250000 2500000 5000000 10000000; do
  python bench.py --config 2 --queries $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sz.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sz.json')); s=d['config']['split_ms']; print($n, round(d['value']/1e6,1), {k: round(v,3) for k,v in s.items()})"
done
