# usage (under gpurun --gpus 2): bash scripts/gpu_fence.sh TAG
TAG=${1:-fe}
mkdir -p gpurun_out
run() {
  for cfg in "toy|--graph --steps 200" "llama3.1-8b|"; do
    wl=${cfg%%|*}; extra=${cfg#*|}
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 \
      bench.py --gpus 2 --workload $wl $extra --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_b.log 2>&1
    grep '^{' gpurun_out/${TAG}_b.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1 $wl $extra', round(d['ms_per_step']*1e3,1), 'us/step')"
  done
}
run fence; run fence
FSDP_B200_NVCC_EXTRA="-DFSDP_HS_NO_FENCE" python -c "import sys; sys.path.insert(0,'paper_2410_06511_b200'); import build; build.build(force=True)" > gpurun_out/${TAG}_build.log 2>&1; echo "rebuild rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu2.log 2>&1; echo "mgpu W=2 (no fence) rc=$?"
run nofence; run nofence
