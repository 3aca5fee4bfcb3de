# usage (under gpurun --gpus N): bash scripts/gpu_store_rs2.sh TAG
TAG=${1:-st}
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p.py -x -q -k "store" > gpurun_out/${TAG}_p2p.log 2>&1; echo "pytest p2p store rc=$?"; tail -1 gpurun_out/${TAG}_p2p.log
for cfg in "store torch" "store library" "pull library"; do set -- $cfg
  for mode in prefetch serial; do flag=""; [ $mode = serial ] && flag="--serial"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus $N --no-e2e --no-cpu-baseline --p2p-rs $1 --grads $2 $flag > gpurun_out/${TAG}_bench_n${N}_$1_$2_$mode.log 2>&1
  grep '^{' gpurun_out/${TAG}_bench_n${N}_$1_$2_$mode.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_serial']
print('rs=$1 grads=$2 $mode', d['ms_per_step'], d['value'], {n: k[n]['GBps'] for n in k if n in ('unshard_push','rs_pull','rs_scatter','rs_reduce','stage_grads')})"
  done
done
