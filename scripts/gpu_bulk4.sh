mkdir -p gpurun_out
FSDP_B200_VARIANT=6 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 \
   tests/mgpu_worker.py > gpurun_out/bulk4_mgpu.log 2>&1; echo "bulk mgpu4 rc=$?"; grep -E "^RANK|Error" gpurun_out/bulk4_mgpu.log | head -5
for v in 0 6; do for g in library torch; do
  FSDP_B200_VARIANT=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --grads $g > gpurun_out/bulk4_v$v_$g.log 2>&1
  grep '^{' gpurun_out/bulk4_v$v_$g.log | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); s=d['kernels_serial']; k=d['kernels']
  print('v=$v grads=$g ms/step', d['ms_per_step'], 'busbw', d['per_rank']['busbw_GBps'], 'serial push', s['unshard_push']['GBps'], 'pull', s['rs_pull']['GBps'])"
done; done
