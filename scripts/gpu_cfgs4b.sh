# usage (under gpurun --gpus 4): bash scripts/gpu_cfgs4b.sh TAG
TAG=${1:-c4b}
mkdir -p gpurun_out
for wl in llama3.1-8b-fp8 llama3.1-70b llama3.1-8b; do for rs in pull store; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus 4 --workload $wl --p2p-rs $rs --grads library --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${wl}_$rs.log 2>&1
  grep '^{' gpurun_out/${TAG}_${wl}_$rs.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_serial']; print('$wl $rs:', d['ms_per_step'], d['value'], {n: k[n]['GBps'] for n in k if n in ('unshard_push','rs_pull','rs_scatter','rs_reduce')})"
done; done
