# usage (under gpurun --gpus 2): bash scripts/gpu_tiles.sh TAG
TAG=${1:-tl}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_property.py -x -q > gpurun_out/${TAG}_p2p.log 2>&1; echo "pytest p2p+property rc=$?"; tail -1 gpurun_out/${TAG}_p2p.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu2.log 2>&1; echo "mgpu W=2 rc=$?"; grep RANK gpurun_out/${TAG}_mgpu2.log
for n in 1 2; do for gflag in "" "--graph"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus $n --workload toy --steps 50 --no-e2e --no-cpu-baseline $gflag > gpurun_out/${TAG}_toy_n${n}${gflag}.log 2>&1
  grep '^{' gpurun_out/${TAG}_toy_n${n}${gflag}.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('toy n=$n $gflag', d['ms_per_step']*1e3, 'us/step', d['value'])"
done; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 \
  scripts/sweep_bench.py --iters 20 --graph --max-log2 22 --out gpurun_out/${TAG}_sweep_w2.jsonl > gpurun_out/${TAG}_sweep.log 2>&1
grep -E 'fsdp_p2p' gpurun_out/${TAG}_sweep_w2.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'log2_bytes' in d: print(d['log2_bytes'], d['unshard_us'], d['rs_us'])"
