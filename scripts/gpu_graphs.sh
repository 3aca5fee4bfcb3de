# usage (under gpurun --gpus 2): bash scripts/gpu_graphs.sh TAG
TAG=${1:-gr}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graphs.py -x -q > gpurun_out/${TAG}_graphs.log 2>&1; echo "pytest graphs rc=$?"; tail -3 gpurun_out/${TAG}_graphs.log
timeout 300 python scripts/graph_probe.py 2>&1 | grep '^{'
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 scripts/graph_probe.py 2>&1 | grep '^{'
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu2.log 2>&1; echo "mgpu W=2 rc=$?"
grep -E "OK|Error|error|assert" gpurun_out/${TAG}_mgpu2.log | head -20
for n in 1 2; do for gflag in "" "--graph"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus $n --workload toy --steps 50 --no-e2e --no-cpu-baseline $gflag > gpurun_out/${TAG}_toy_n${n}${gflag}.log 2>&1
  echo "toy n=$n $gflag rc=$?"; grep '^{' gpurun_out/${TAG}_toy_n${n}${gflag}.log | tail -1 | cut -c1-200
done; done
