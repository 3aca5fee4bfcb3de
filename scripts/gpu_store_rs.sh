# usage (under gpurun --gpus N): bash scripts/gpu_store_rs.sh TAG
TAG=${1:-st}
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p.py -x -q -k "store or pull" > gpurun_out/${TAG}_p2p.log 2>&1; echo "pytest p2p rc=$?"; tail -1 gpurun_out/${TAG}_p2p.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu$N.log 2>&1; echo "mgpu W=$N rc=$?"
grep -E "RANK|mode|Error|error|assert" gpurun_out/${TAG}_mgpu$N.log | head -12
for rs in store pull; do for gr in torch library; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus $N --no-e2e --no-cpu-baseline --p2p-rs $rs --grads $gr > gpurun_out/${TAG}_bench_n${N}_${rs}_${gr}.log 2>&1
  grep '^{' gpurun_out/${TAG}_bench_n${N}_${rs}_${gr}.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_serial']
print('rs=$rs grads=$gr', d['ms_per_step'], d['value'], {n: k[n]['GBps'] for n in k if n in ('unshard_push','rs_pull','rs_scatter','rs_reduce','stage_grads')}, d['roofline']['kernel'], d['roofline']['frac'])"
done; done
