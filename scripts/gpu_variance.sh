# usage (under gpurun --gpus 4): bash scripts/gpu_variance.sh TAG — default bench lines, repeated
TAG=${1:-var}
mkdir -p gpurun_out
for i in 1 2; do for n in 1 2 4; do
  if [ $n = 1 ]; then timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_n${n}_$i.log 2>&1
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29556 \
         bench.py --gpus $n > gpurun_out/${TAG}_n${n}_$i.log 2>&1; fi
  grep '^{' gpurun_out/${TAG}_n${n}_$i.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('run $i n=$n', d['ms_per_step'], d['value'], d['ms_per_step_pct'], 'e2e', d['e2e']['value'] if d.get('e2e') else None, d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
