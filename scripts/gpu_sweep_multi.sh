N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
for n in 2 4; do
  [ $n -gt $N ] && continue
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29557 \
    scripts/sweep_bench.py --out gpurun_out/sweep_w$n.jsonl > gpurun_out/sweep_w$n.log 2>&1; echo "w=$n rc=$?"
done
