# usage (under gpurun --gpus 2): bash scripts/gpu_pullsweep.sh TAG
TAG=${1:-ps}
mkdir -p gpurun_out
for cfg in "4096 2" "16384 4" "8192 3"; do
  set -- $cfg
  FSDP_B200_PULL_CHUNK=$1 FSDP_B200_PULL_STAGES=$2 timeout 600 python -m pytest tests/test_gpu_p2p.py -x -q \
    > gpurun_out/${TAG}_p2p_$1_$2.log 2>&1; echo "p2p parity chunk=$1 stages=$2 rc=$?"; tail -1 gpurun_out/${TAG}_p2p_$1_$2.log
done
FSDP_B200_PULL_CHUNK=16384 FSDP_B200_PULL_STAGES=4 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29555 tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu2.log 2>&1; echo "mgpu W=2 (16K,4) rc=$?"
for cfg in "4096 2" "4096 3" "4096 4" "8192 2" "8192 3" "8192 4" "16384 2" "16384 3"; do
  set -- $cfg
  FSDP_B200_PULL_CHUNK=$1 FSDP_B200_PULL_STAGES=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --no-e2e --no-cpu-baseline \
    > gpurun_out/${TAG}_bench_$1_$2.log 2>&1
  grep '^{' gpurun_out/${TAG}_bench_$1_$2.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_serial']
print('chunk=$1 stages=$2', d['ms_per_step'], d['value'], 'pull', k.get('rs_pull',{}).get('GBps'), 'push', k.get('unshard_push',{}).get('GBps'))"
done
