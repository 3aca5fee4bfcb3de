# Round 2 on 4 GPUs: multi-GPU worker (W=4, W=2), HSDP 2x2 / 4x1 (gather on the second
# stream), FSDP-4 bf16 / fp8 delayed / fp8 dynamic / 70B, N=2 bf16 (under gpurun --gpus 4)
O=gpurun_out/${1:-r2n4}
mkdir -p $O
timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -2 $O/pytest_mgpu.log
B="python bench.py --no-cpu-baseline --no-e2e --out $O/bench.jsonl"
timeout 600 $B --gpus 4 --shard-size 2 > $O/b_hsdp22.log 2>&1; echo "hsdp 2x2 rc=$?"
timeout 600 $B --gpus 4 --shard-size 1 > $O/b_hsdp41.log 2>&1; echo "hsdp 4x1 rc=$?"
timeout 600 $B --gpus 4 > $O/b_n4.log 2>&1; echo "n4 rc=$?"
timeout 600 $B --gpus 4 --workload llama3.1-8b-fp8 --fp8-scaling delayed > $O/b_n4_fp8d.log 2>&1; echo "n4 fp8 delayed rc=$?"
timeout 600 $B --gpus 4 --workload llama3.1-8b-fp8 > $O/b_n4_fp8.log 2>&1; echo "n4 fp8 dynamic rc=$?"
timeout 600 $B --gpus 4 --workload llama3.1-70b > $O/b_n4_70b.log 2>&1; echo "n4 70b rc=$?"
timeout 600 $B --gpus 2 > $O/b_n2.log 2>&1; echo "n2 rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["config"]["shard_size"], d["ms_per_step"], d["config"]["workload"][:16], d["config"]["collectives"][-50:], (d.get("wire") or {}).get("GBps_per_direction"), d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
