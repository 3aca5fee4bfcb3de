# full validation on the GPUs of this box: smoke, all GPU tests (multi-GPU test runs on every visible GPU), benches
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench n1 rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-400
if [ $N -ge 2 ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 \
   bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "bench n$N rc=$?"; grep '^{' gpurun_out/bench_n$N.log | cut -c1-400
fi
