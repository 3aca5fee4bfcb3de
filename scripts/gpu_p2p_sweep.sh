# under gpurun --gpus 2: correctness of the pull variant, then push/pull NVLink GB/s vs variant and CTAs/SM
mkdir -p gpurun_out
FSDP_B200_VARIANT=1 timeout 900 python -m pytest tests/test_gpu_p2p.py -q -x -k "pull" > gpurun_out/sw_p2p_tests.log 2>&1; echo "vec8 pull tests rc=$?"; tail -2 gpurun_out/sw_p2p_tests.log
for v in 0 1; do for c in 0 2 4 8; do
  env FSDP_B200_VARIANT=$v $( [ $c -gt 0 ] && echo FSDP_B200_CTAS_PER_SM=$c ) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --steps 3 --warmup 2 --no-e2e > gpurun_out/sw_v${v}_c${c}.log 2>&1
  grep '^{' gpurun_out/sw_v${v}_c${c}.log | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); s=d['kernels_serial']
  print('v=$v c=$c ms/step', d['ms_per_step'], 'push', s['unshard_push']['GBps'], 'pull', s['rs_pull']['GBps'])"
done; done
