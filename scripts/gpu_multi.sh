# usage (under gpurun --gpus N): bash scripts/gpu_multi.sh TAG [algos] [modes]
TAG=${1:-m}
ALGOS=${2:-"p2p nccl"}
MODES=${3:-"prefetch serial"}
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/${TAG}_topo.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu.log 2>&1; echo "mgpu rc=$?"; grep -E "OK|Error|error|assert" gpurun_out/${TAG}_mgpu.log | head -20
for n in $(seq 2 $N); do
  case $n in 2|4|8) ;; *) continue;; esac
  for algo in $ALGOS; do for mode in $MODES; do
  flag=""; [ "$mode" = serial ] && flag="--serial"
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
     bench.py --gpus $n --steps 5 --warmup 3 --no-e2e --algo $algo $flag > gpurun_out/${TAG}_bench_n${n}_${algo}_${mode}.log 2>&1
  echo "bench n=$n $algo $mode rc=$?"; grep '^{' gpurun_out/${TAG}_bench_n${n}_${algo}_${mode}.log | tail -1 | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); k=d['kernels']
  print('  ms/step', d['ms_per_step'], 'value', d['value'], 'busbw/rank', d['per_rank']['busbw_GBps'], 'frac', d['per_rank']['busbw_frac_nvlink_900'], 'roofline', d['roofline']['kernel'], d['roofline']['frac'])
  print('  ', {n: (v['avg_us'], v['GBps']) for n, v in k.items()})
"
  done; done
done
