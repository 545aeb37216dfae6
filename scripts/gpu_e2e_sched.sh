# host-buffer pipeline: chunk schedule sweep (P2M_E2E_SCHED = first,growth,cap,tail as fractions of the batch)
for sch in "0.03125,2,0.25,0" "0.05,2,0.25,0.05" "0.05,3,0.4,0.1" "0.05,2,0.4,0" "0.1,2,0.4,0" "0.0625,1.5,0.3,0.05" "0.03125,2,0.25,0.0625" "0.1,1,0.1,0" "0.125,2,0.5,0" "0.02,2,0.2,0.02"; do
  for cfg in 2 1; do
    P2M_E2E_SCHED=$sch python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 6 > gpurun_out/sch.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/sch.json')); print('$sch c$cfg e2e', round(d['e2e']['value']/1e6,1), d['e2e']['rows_equal_device_path'])"
  done
done
