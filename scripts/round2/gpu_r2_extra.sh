# Round 2 extra configs on 4 GPUs: HSDP 2x2 with fp8 (delayed), HSDP 2x2 train step, FSDP-4
# train / zero2, fp8 delayed N=2, toy graph N=1/2/4 with the queued-start timing
O=gpurun_out/${1:-r2extra}
mkdir -p $O
B="python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl"
timeout 600 $B --gpus 4 --shard-size 2 --workload llama3.1-8b-fp8 --fp8-scaling delayed > $O/b1.log 2>&1; echo "hsdp fp8 rc=$?"
timeout 600 $B --gpus 4 --shard-size 2 --step train > $O/b2.log 2>&1; echo "hsdp train rc=$?"
timeout 600 $B --gpus 4 --step train > $O/b3.log 2>&1; echo "fsdp4 train rc=$?"
timeout 600 $B --gpus 4 --step train --zero2 > $O/b4.log 2>&1; echo "fsdp4 zero2 rc=$?"
timeout 600 $B --gpus 2 --workload llama3.1-8b-fp8 --fp8-scaling delayed > $O/b5.log 2>&1; echo "n2 fp8 delayed rc=$?"
for n in 1 2 4; do timeout 600 $B --gpus $n --workload toy --graph --steps 200 --warmup 20 > $O/toy_n$n.log 2>&1; echo "toy graph n$n rc=$?"; done
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    c = d["config"]
    print(d["n_gpus"], c["shard_size"], c["step"], d["ms_per_step"], c["workload"][:30], (d.get("wire") or {}).get("GBps_per_direction"), d["isolated"]["ms_per_step"])
PY
