# usage (under gpurun --gpus 4): bash scripts/gpu_auto_small.sh TAG
TAG=${1:-as}
mkdir -p gpurun_out
for rs in ${RS:-auto store}; do for cfg in "toy|--graph --steps 200" "llama3.1-8b|"; do
  wl=${cfg%%|*}; extra=${cfg#*|}
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus 4 --workload $wl $extra --p2p-rs $rs --grads library --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_b.log 2>&1
  grep '^{' gpurun_out/${TAG}_b.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('rs=$rs $wl $extra', round(d['ms_per_step']*1e3,1), 'us/step', d['value'])"
done; done
[ -n "$SKIP_WORKER" ] || timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu4.log 2>&1; echo "mgpu W=4 rc=$?"; grep RANK gpurun_out/${TAG}_mgpu4.log
