mkdir -p gpurun_out
run() {
  name=$1; n=$2; shift 2
  if [ $n = 1 ]; then timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/cfg_${name}.log 2>&1
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
     bench.py --gpus $n --steps 10 --warmup 3 --no-e2e "$@" > gpurun_out/cfg_${name}.log 2>&1; fi
  echo "$name rc=$?"; grep '^{' gpurun_out/cfg_${name}.log | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); r=d['roofline']
  print('  ms/step', d['ms_per_step'], 'value', d['value'], 'busbw/rank', d['per_rank']['busbw_GBps'], 'frac', d['per_rank']['busbw_frac_nvlink_900'], '| roofline', r['kernel'], r['achieved'], r['frac'])
  print('   serial', {k:(v['avg_us'],v['GBps']) for k,v in d['kernels_serial'].items()})"
}
run toy_n1 1 --workload toy
run toy_n2 2 --workload toy
run toy_n4 4 --workload toy
run l70_n4 4 --workload llama3.1-70b
run fp8_n4 4 --workload llama3.1-8b-fp8
run fp8_n1 1 --workload llama3.1-8b-fp8
run l8_n4 4
run l8_n4_train 4 --step train
