mkdir -p gpurun_out
FSDP_B200_VARIANT=14 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x -k "rs_copy_in or full_path or tails" > gpurun_out/k5b_tests.log 2>&1; echo "k5 bulk tests rc=$?"; tail -1 gpurun_out/k5b_tests.log
for v in 6 14; do
  FSDP_B200_VARIANT=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k5b.log 2>&1
  grep '^{' gpurun_out/k5b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('v=$v ms/step', d['ms_per_step'], 'value', d['value'], 'step_hbm', r['step_hbm_frac'], {k:(v['avg_us'],v['GBps']) for k,v in d['kernels_serial'].items()})"
done
