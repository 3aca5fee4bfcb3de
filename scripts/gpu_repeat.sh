# usage (under gpurun --gpus 4): bash scripts/gpu_repeat.sh TAG — repeated multi-GPU parity runs
TAG=${1:-rp}
mkdir -p gpurun_out
for i in 1 2 3; do for n in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n \
     tests/mgpu_worker.py > gpurun_out/${TAG}_w${n}_$i.log 2>&1; rc=$?
  echo "run $i W=$n rc=$rc OK-lines=$(grep -c 'OK' gpurun_out/${TAG}_w${n}_$i.log)"
  if [ $rc != 0 ]; then grep -E "Error|assert" gpurun_out/${TAG}_w${n}_$i.log | head -5; fi
done; done
