# usage (under gpurun --gpus 4): bash scripts/gpu_store_rs4.sh TAG
TAG=${1:-st4}
N=4
mkdir -p gpurun_out
for cfg in "store torch" "store library" "pull library" "pull torch"; do set -- $cfg
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus $N --no-e2e --no-cpu-baseline --p2p-rs $1 --grads $2 > gpurun_out/${TAG}_bench_n${N}_$1_$2.log 2>&1
  grep '^{' gpurun_out/${TAG}_bench_n${N}_$1_$2.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_serial']
print('rs=$1 grads=$2', d['ms_per_step'], d['value'], {n: k[n]['GBps'] for n in k if n in ('unshard_push','rs_pull','rs_scatter','rs_reduce','stage_grads')})"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29557 \
    bench.py --gpus 3 --no-e2e --no-cpu-baseline --p2p-rs store --grads torch > gpurun_out/${TAG}_bench_n3_store.log 2>&1
grep '^{' gpurun_out/${TAG}_bench_n3_store.log | cut -c1-150
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29557 \
    bench.py --gpus 3 --no-e2e --no-cpu-baseline --p2p-rs pull --grads library > gpurun_out/${TAG}_bench_n3_pull.log 2>&1
grep '^{' gpurun_out/${TAG}_bench_n3_pull.log | cut -c1-150
