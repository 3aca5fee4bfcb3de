# every -m gpu test on the box's GPUs + smoke (after a refactor)
O=gpurun_out/${1:-r2tests}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log | cut -c1-120
timeout 2700 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/b_n2.log 2>&1; echo "n2 rc=$?"; grep '^{' $O/b_n2.log | cut -c1-200
