# usage (under gpurun --gpus 4): bash scripts/gpu_ctas.sh TAG
TAG=${1:-ct}
mkdir -p gpurun_out
for n in 4 2; do for c in 0 2 3 4; do
  env_c=""; [ $c != 0 ] && env_c="FSDP_B200_CTAS_PER_SM=$c"
  env $env_c timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus $n --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_n${n}_c$c.log 2>&1
  grep '^{' gpurun_out/${TAG}_n${n}_c$c.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_serial']; print('n=$n ctas_per_sm=$c', d['ms_per_step'], d['value'], {n: k[n]['GBps'] for n in k if n in ('unshard_push','rs_scatter','rs_pull','rs_reduce')})"
done; done
