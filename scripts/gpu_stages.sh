# usage (under gpurun, 1 GPU): bash scripts/gpu_stages.sh TAG
TAG=${1:-st}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python scripts/stage_bench.py --out gpurun_out/${TAG}_stages_8b.jsonl > gpurun_out/${TAG}_stages_8b.log 2>&1
echo "stage_bench 8b rc=$?"
timeout 900 python scripts/stage_bench.py --model llama3.1-70b --ws 1,8 --no-torch --iters 10 \
  --out gpurun_out/${TAG}_stages_70b.jsonl > gpurun_out/${TAG}_stages_70b.log 2>&1
echo "stage_bench 70b rc=$?"
