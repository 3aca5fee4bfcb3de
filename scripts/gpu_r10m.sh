# usage (under gpurun --gpus 4): bash scripts/gpu_r10m.sh TAG
TAG=${1:-r10m}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/${TAG}_multigpu.log 2>&1; echo "pytest multigpu rc=$?"
tail -2 gpurun_out/${TAG}_multigpu.log
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
   bench.py --gpus $n > gpurun_out/${TAG}_bench_n$n.log 2>&1; echo "bench n=$n rc=$?"
grep '^{' gpurun_out/${TAG}_bench_n$n.log | tail -1 | cut -c1-300
done
