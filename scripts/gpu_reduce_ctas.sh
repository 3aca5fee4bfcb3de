# usage (under gpurun --gpus 4): bash scripts/gpu_reduce_ctas.sh TAG
TAG=${1:-rc}
mkdir -p gpurun_out
for wl in llama3.1-8b-fp8 llama3.1-8b; do for rc in 0 1 2; do
  FSDP_B200_REDUCE_CTAS_PER_SM=$rc timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus 4 --workload $wl --p2p-rs store --grads library --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${wl}_rc$rc.log 2>&1
  grep '^{' gpurun_out/${TAG}_${wl}_rc$rc.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']; print('$wl reduce_ctas=$rc', d['ms_per_step'], d['value'], {n: (k[n]['avg_us'], k[n]['share_of_step']) for n in k if n in ('unshard_push','rs_scatter','rs_reduce')})"
done; done
