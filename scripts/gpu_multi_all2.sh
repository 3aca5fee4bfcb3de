# usage (under gpurun --gpus 4): bash scripts/gpu_multi_all2.sh TAG
TAG=${1:-ma}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/${TAG}_multigpu.log 2>&1; echo "pytest multigpu rc=$?"
tail -2 gpurun_out/${TAG}_multigpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu3.log 2>&1; echo "mgpu W=3 rc=$?"
grep -E "RANK|mode|Error|error|assert" gpurun_out/${TAG}_mgpu3.log | head -8
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
   bench.py --gpus $n > gpurun_out/${TAG}_bench_n$n.log 2>&1; echo "bench n=$n rc=$?"
grep '^{' gpurun_out/${TAG}_bench_n$n.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['config']['collectives'], d['config']['grads'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline'].get('sm_mechanism_ceiling'), 'e2e', d['e2e']['value'] if d.get('e2e') else None)"
done
