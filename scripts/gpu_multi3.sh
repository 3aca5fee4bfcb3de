# under gpurun --gpus N: parity worker, then P2P bench with library (zero-copy) vs torch grads
TAG=${1:-z}
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu.log 2>&1; echo "mgpu rc=$?"; grep -E "^RANK|Error|error|assert" gpurun_out/${TAG}_mgpu.log | sort | uniq | head -20
run() {
  name=$1; n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
     bench.py --gpus $n --steps 5 --warmup 3 "$@" > gpurun_out/${TAG}_${name}.log 2>&1
  echo "bench $name rc=$?"; grep '^{' gpurun_out/${TAG}_${name}.log | tail -1 | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); r=d['roofline']
  print('  ms/step', d['ms_per_step'], 'value', d['value'], 'busbw/rank', d['per_rank']['busbw_GBps'], 'frac', d['per_rank']['busbw_frac_nvlink_900'], '| roofline', r['kernel'], r['achieved'], r['frac'], '| e2e', (d['e2e'] or {}).get('value'))
  print('   step', {k:(v['avg_us'],v['GBps']) for k,v in d['kernels'].items()})
  print('   serial', {k:(v['avg_us'],v['GBps']) for k,v in d['kernels_serial'].items()})
"
  grep -E "Error|error" gpurun_out/${TAG}_${name}.log | head -3
}
run n${N}_lib $N
run n${N}_torch $N --grads torch --no-e2e
