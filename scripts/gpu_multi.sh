# usage (under gpurun --gpus N): bash scripts/gpu_multi.sh TAG
TAG=${1:-m}
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/${TAG}_topo.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu.log 2>&1; echo "mgpu rc=$?"; grep -E "OK|Error|error" gpurun_out/${TAG}_mgpu.log | head -20
for n in $(seq 2 $N); do
  case $n in 2|4|8) ;; *) continue;; esac
  for mode in "" "--serial"; do
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
     bench.py --gpus $n --steps 5 --warmup 3 --no-e2e $mode > gpurun_out/${TAG}_bench_n${n}${mode}.log 2>&1
  echo "bench n=$n $mode rc=$?"; grep '^{' gpurun_out/${TAG}_bench_n${n}${mode}.log | tail -1
  done
done
