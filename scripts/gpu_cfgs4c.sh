# usage (under gpurun --gpus 4): bash scripts/gpu_cfgs4c.sh TAG
TAG=${1:-c4c}
mkdir -p gpurun_out
for cfg in "llama3.1-8b-fp8|" "llama3.1-70b|" "llama3.1-8b|--step train" "llama3.1-8b|--step train --zero2" "llama3.1-8b|--shard-size 2" "toy|--graph --steps 50" "toy|--steps 50"; do
  wl=${cfg%%|*}; extra=${cfg#*|}; name=$(echo "$wl $extra" | tr ' -' '__')
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 \
    bench.py --gpus 4 --workload $wl $extra --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_$name.log 2>&1
  grep '^{' gpurun_out/${TAG}_$name.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$wl $extra:', d['ms_per_step'], d['value'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])"
done
