# under gpurun --gpus 4: parity worker (P2P + NCCL + HSDP) and benches of the step variants
TAG=${1:-q}
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu.log 2>&1; echo "mgpu rc=$?"; grep -E "OK|Error|error|assert" gpurun_out/${TAG}_mgpu.log | sort | uniq | head -30
run() {  # name n args...
  name=$1; n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
     bench.py --gpus $n --steps 5 --warmup 3 --no-e2e "$@" > gpurun_out/${TAG}_${name}.log 2>&1
  echo "bench $name rc=$?"; grep '^{' gpurun_out/${TAG}_${name}.log | tail -1 | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); r=d['roofline']
  print('  ms/step', d['ms_per_step'], 'value', d['value'], 'busbw/rank', d['per_rank']['busbw_GBps'], 'frac', d['per_rank']['busbw_frac_nvlink_900'], '| roofline', r['kernel'], r['achieved'], r['frac'])
  print('   step', {k:(v['avg_us'],v['GBps']) for k,v in d['kernels'].items()})
  print('   serial', {k:(v['avg_us'],v['GBps']) for k,v in d['kernels_serial'].items()})
"
  grep -E "Error|error" gpurun_out/${TAG}_${name}.log | head -3
}
run n${N}_p2p $N
run n${N}_nccl $N --algo nccl
run n${N}_train $N --step train
run n${N}_hsdp2 $N --shard-size 2
run n2_p2p 2
