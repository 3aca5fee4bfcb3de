# usage (under gpurun, 1 GPU): bash scripts/gpu_w1k2.sh TAG
TAG=${1:-k2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py tests/test_gpu_training_step.py tests/test_gpu_guards.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
for v in 14 46 14 46; do
  FSDP_B200_VARIANT=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_v$v.log 2>&1
  grep '^{' gpurun_out/${TAG}_bench_v$v.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_serial']; print('variant $v', d['ms_per_step'], d['value'], {n: k[n]['GBps'] for n in k}, d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['step_hbm_frac'])"
done
