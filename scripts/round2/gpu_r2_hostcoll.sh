# Round 2: host-collective mesh, N processes on ONE GPU (cross-process P2P protocol), plus
# the multi-GPU worker (P2P amax all-reduce) when more GPUs are visible
O=gpurun_out/${1:-r2hc}
mkdir -p $O
N=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  P=$(python -c "import socket;s=socket.socket();s.bind(('127.0.0.1',0));print(s.getsockname()[1])")
  CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 \
    --master-port $P tests/hostcoll_worker.py > $O/hostcoll_n$n.log 2>&1; echo "hostcoll n$n rc=$?"; grep -c "hostcoll OK" $O/hostcoll_n$n.log; tail -3 $O/hostcoll_n$n.log | cut -c1-300
done
if [ $N -ge 2 ]; then
  timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -2 $O/pytest_mgpu.log
  timeout 600 python bench.py --gpus 2 --workload llama3.1-8b-fp8 --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/b_n2_fp8.log 2>&1; echo "n2 fp8 rc=$?"
fi
