mkdir -p gpurun_out
for b in 0 1; do
  env $( [ $b = 1 ] && echo FSDP_B200_W1_BULK=1 ) timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/w1b.log 2>&1
  grep '^{' gpurun_out/w1b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('w1bulk=$b ms/step', d['ms_per_step'], 'value', d['value'], 'step_hbm', r['step_hbm_frac'], {k:(v['avg_us'],v['GBps']) for k,v in d['kernels_serial'].items()})"
done
