# usage (under gpurun --gpus 2): bash scripts/gpu_pdl.sh TAG
TAG=${1:-pd}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_property.py tests/test_gpu_graphs.py -x -q > gpurun_out/${TAG}_p2p.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_p2p.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/${TAG}_mgpu2.log 2>&1; echo "mgpu W=2 rc=$?"; grep -c "OK" gpurun_out/${TAG}_mgpu2.log; grep -E "Error|assert" gpurun_out/${TAG}_mgpu2.log | head -3
for pdl in 1 0 1 0; do for cfg in "toy|--graph --steps 100" "toy|--steps 100" "llama3.1-8b|"; do
  wl=${cfg%%|*}; extra=${cfg#*|}
  FSDP_B200_PDL=$pdl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus 2 --workload $wl $extra --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_b.log 2>&1
  grep '^{' gpurun_out/${TAG}_b.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('pdl=$pdl $wl $extra', round(d['ms_per_step']*1e3,1), 'us/step')"
done; done
