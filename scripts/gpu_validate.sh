# Validation on the GPUs of this box: smoke, all GPU tests (the multi-GPU test runs on
# every visible GPU), bench at N=1 and N=all, launch list of the N=1 bench under ncu.
# usage (under gpurun [--gpus N]): bash scripts/gpu_validate.sh TAG
TAG=${1:-val}
O=gpurun_out/$TAG
mkdir -p $O
N=$(nvidia-smi -L | wc -l)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpus.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py --out $O/bench.jsonl > $O/bench_n1.log 2>&1; echo "bench n1 rc=$?"; tail -1 $O/bench_n1.log | cut -c1-300
if [ $N -ge 2 ]; then
timeout 900 python bench.py --gpus $N --out $O/bench.jsonl > $O/bench_n$N.log 2>&1; echo "bench n$N rc=$?"; grep '^{' $O/bench_n$N.log | cut -c1-300
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 600 --csv --log-file $O/launches_w1.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu rc=$?"
