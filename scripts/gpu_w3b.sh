# usage (under gpurun --gpus 4): bash scripts/gpu_w3b.sh TAG
TAG=${1:-w3}
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu3.log 2>&1; echo "mgpu W=3 rc=$?"
grep -E "OK|Error|error|assert" gpurun_out/${TAG}_mgpu3.log | head -30
for n in 4 3; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
   bench.py --gpus $n > gpurun_out/${TAG}_bench_n$n.log 2>&1; echo "bench n=$n rc=$?"
grep '^{' gpurun_out/${TAG}_bench_n$n.log | tail -1 | cut -c1-420
done
