# Round 2 last 4-GPU refresh of the final code: N=2 / N=4 / HSDP 2x2 / fp8 delayed N=4 /
# 70B N=1 benches, and one ncu --set full capture of the W=1 TMA cast (under gpurun --gpus 4)
O=gpurun_out/${1:-r2last}
mkdir -p $O
B="python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl"
timeout 600 $B --gpus 2 > $O/b_n2.log 2>&1; echo "n2 rc=$?"
timeout 600 $B --gpus 4 > $O/b_n4.log 2>&1; echo "n4 rc=$?"
timeout 600 $B --gpus 4 --shard-size 2 > $O/b_hsdp.log 2>&1; echo "hsdp rc=$?"
timeout 600 $B --gpus 4 --workload llama3.1-8b-fp8 --fp8-scaling delayed > $O/b_fp8.log 2>&1; echo "fp8 n4 rc=$?"
timeout 600 $B --workload llama3.1-70b > $O/b_70b.log 2>&1; echo "70b n1 rc=$?"
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_cast_w1" -s 40 -c 1 -o $O/prof_cast $C > $O/ncu_cast.log 2>&1; echo "ncu cast rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["config"]["shard_size"], d["config"]["workload"][:16], d["ms_per_step"], d["ms_per_step_pct"]["median"], (d.get("wire") or {}).get("GBps_per_direction"), d["roofline"]["kernel"], d["roofline"]["frac"])
PY
