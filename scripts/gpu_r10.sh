# usage (under gpurun, 1 GPU): bash scripts/gpu_r10.sh TAG
TAG=${1:-r10}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest gpu rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python scripts/stage_bench.py --out gpurun_out/${TAG}_stages_8b.jsonl > gpurun_out/${TAG}_stages_8b.log 2>&1
echo "stage_bench 8b rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_n1.log 2>&1; echo "bench n1 rc=$?"
grep '^{' gpurun_out/${TAG}_bench_n1.log | tail -1 | cut -c1-300
timeout 900 python bench.py --workload llama3.1-8b-fp8 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_fp8_n1.log 2>&1
echo "bench fp8 n1 rc=$?"
