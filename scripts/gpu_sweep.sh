# 1-GPU tuning sweep: CTAs per SM for the HBM kernels, plus the fp8 and 70B workloads
mkdir -p gpurun_out
for c in 2 4 6 8; do
  FSDP_B200_CTAS_PER_SM=$c timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --serial > gpurun_out/sweep_c$c.log 2>&1
  echo "ctas/sm=$c rc=$?"; grep '^{' gpurun_out/sweep_c$c.log | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); print('  ms/step', d['ms_per_step'], {k:(v['avg_us'],v['GBps']) for k,v in d['kernels'].items()})"
done
for wl in llama3.1-8b-fp8 llama3.1-70b; do
  timeout 900 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --workload $wl > gpurun_out/sweep_$wl.log 2>&1
  echo "$wl rc=$?"; grep '^{' gpurun_out/sweep_$wl.log | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); print('  ms/step', d['ms_per_step'], 'value', d['value'], {k:(v['avg_us'],v['GBps']) for k,v in d['kernels'].items()})"
done
