# usage (under gpurun --gpus 4): bash scripts/gpu_sweep_graph.sh TAG
TAG=${1:-swg}
mkdir -p gpurun_out
for n in 4 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n \
  scripts/sweep_bench.py --iters 20 --graph --out gpurun_out/${TAG}_sweep_w$n.jsonl > gpurun_out/${TAG}_sweep_w$n.log 2>&1
echo "sweep graph W=$n rc=$?"; grep alpha_B gpurun_out/${TAG}_sweep_w$n.jsonl; grep -E '"log2_bytes": (16|20),' gpurun_out/${TAG}_sweep_w$n.jsonl | cut -c1-200
done
