mkdir -p gpurun_out
for cfg in "" "FSDP_B200_CTAS_PER_SM=4"; do for mode in "" "--serial"; do
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $mode > gpurun_out/w1m.log 2>&1
  grep '^{' gpurun_out/w1m.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('cfg=[$cfg] mode=[$mode] ms/step', d['ms_per_step'], 'value', d['value'], 'step_hbm_frac', r['step_hbm_frac'], {k:(v['avg_us'],v['GBps']) for k,v in d['kernels_serial'].items()})"
done; done
