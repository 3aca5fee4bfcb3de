mkdir -p gpurun_out
FSDP_B200_VARIANT=6 timeout 900 python -m pytest tests/test_gpu_p2p.py -q -x > gpurun_out/bulk_tests.log 2>&1; echo "bulk emulated tests rc=$?"; tail -1 gpurun_out/bulk_tests.log
FSDP_B200_VARIANT=6 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/bulk_mgpu.log 2>&1; echo "bulk mgpu rc=$?"; grep -E "^RANK|Error" gpurun_out/bulk_mgpu.log | head -4
for v in 0 2 4 6; do
  FSDP_B200_VARIANT=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bulk_v$v.log 2>&1
  grep '^{' gpurun_out/bulk_v$v.log | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); s=d['kernels_serial']; k=d['kernels']
  print('v=$v ms/step', d['ms_per_step'], 'serial push', s['unshard_push']['GBps'], 'pull', s['rs_pull']['GBps'], '| in-step push', k['unshard_push']['GBps'], 'pull', k['rs_pull']['GBps'])"
done
