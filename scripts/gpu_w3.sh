# usage (under gpurun --gpus 4): bash scripts/gpu_w3.sh TAG
# Non-power-of-two world (W=3): parity worker, then the 2/4-GPU pytest.
TAG=${1:-w3}
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu3.log 2>&1; echo "mgpu W=3 rc=$?"
grep -E "OK|Error|error|assert" gpurun_out/${TAG}_mgpu3.log | head -20
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/${TAG}_multigpu.log 2>&1; echo "pytest multigpu rc=$?"
tail -3 gpurun_out/${TAG}_multigpu.log
