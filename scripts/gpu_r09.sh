# usage (under gpurun, 1 GPU): bash scripts/gpu_r09.sh TAG
TAG=${1:-r09}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest gpu rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python scripts/stage_bench.py --out gpurun_out/${TAG}_stages_8b.jsonl > gpurun_out/${TAG}_stages_8b.log 2>&1
echo "stage_bench 8b rc=$?"
timeout 900 python scripts/stage_bench.py --model llama3.1-70b --ws 1,8 --no-torch --iters 10 \
  --out gpurun_out/${TAG}_stages_70b.jsonl > gpurun_out/${TAG}_stages_70b.log 2>&1
echo "stage_bench 70b rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_n1.log 2>&1; echo "bench n1 rc=$?"
tail -1 gpurun_out/${TAG}_bench_n1.log | cut -c1-600
timeout 900 python bench.py --workload llama3.1-70b --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_70b.log 2>&1
echo "bench 70b rc=$?"
timeout 900 python bench.py --workload llama3.1-70b --no-e2e --no-cpu-baseline --compute-tokens 4096 \
  > gpurun_out/${TAG}_bench_70b_proxy.log 2>&1; echo "bench 70b proxy rc=$?"
grep -o '"compute_proxy": {[^}]*}' gpurun_out/${TAG}_bench_70b_proxy.log
