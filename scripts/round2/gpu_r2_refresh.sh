# Round 2 refresh on 4 GPUs: N=1 (8-CTA bf16 push) x2, 70B N=1/2, toy graph N=1/2/4, ragged
# sweep + alpha-B fit at W=2 and W=4 (under gpurun --gpus 4)
O=gpurun_out/${1:-r2refresh}
mkdir -p $O
B="python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl"
for i in 1 2; do timeout 600 $B > $O/b_n1_$i.log 2>&1; echo "n1 rc=$?"; done
timeout 600 $B --workload llama3.1-70b > $O/b_70b_n1.log 2>&1; echo "70b n1 rc=$?"
timeout 600 $B --gpus 2 --workload llama3.1-70b > $O/b_70b_n2.log 2>&1; echo "70b n2 rc=$?"
for n in 1 2 4; do timeout 600 $B --gpus $n --workload toy --graph --steps 200 --warmup 20 > $O/b_toy_n$n.log 2>&1; echo "toy graph n$n rc=$?"; done
for n in 2 4; do
  P=$(python -c "import socket;s=socket.socket();s.bind(('127.0.0.1',0));print(s.getsockname()[1])")
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port $P \
    scripts/sweep_bench.py --out $O/sweep_w$n.jsonl > $O/sweep_w$n.log 2>&1; echo "sweep w$n rc=$?"
  grep alpha_B $O/sweep_w$n.jsonl | cut -c1-200
done
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["ms_per_step"], d["config"]["workload"][:24], d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()}, d["roofline"]["frac"], d["roofline"].get("step_hbm_frac"))
PY
