# usage (under gpurun --gpus 4): bash scripts/gpu_reduce_ctas2.sh TAG
TAG=${1:-rc}
mkdir -p gpurun_out
for n in 4 2; do for wl in llama3.1-8b-fp8 llama3.1-8b; do for cfg in "store 3" "store 2" "pull 2"; do set -- $cfg
  FSDP_B200_REDUCE_CTAS_PER_SM=$2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus $n --workload $wl --p2p-rs $1 --grads library --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_n${n}_${wl}_$1_rc$2.log 2>&1
  grep '^{' gpurun_out/${TAG}_n${n}_${wl}_$1_rc$2.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('n=$n $wl rs=$1 reduce_ctas=$2', d['ms_per_step'], d['value'])"
done; done; done
