# usage (under gpurun --gpus 4): bash scripts/gpu_multi_only.sh TAG
TAG=${1:-mo}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/${TAG}_multigpu.log 2>&1; echo "pytest multigpu rc=$?"; tail -2 gpurun_out/${TAG}_multigpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu3.log 2>&1; echo "mgpu W=3 rc=$?"
grep -E "RANK|full-size|Error|assert" gpurun_out/${TAG}_mgpu3.log | head -8
