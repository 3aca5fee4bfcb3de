# Round 2: after the push/K3 register fix (amax as a template parameter) and the sticky
# abort reason: multi-GPU worker at W=2, benches at N=1 (bf16, fp8 delayed/dynamic) and N=2,
# the copy-engine path at N=2.
O=gpurun_out/${1:-r2fix}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -2 $O/pytest_mgpu.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/bench_n1.log 2>&1; echo "bench n1 rc=$?"
for sc in delayed dynamic; do
timeout 600 python bench.py --workload llama3.1-8b-fp8 --fp8-scaling $sc --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/bench_fp8_$sc.log 2>&1; echo "bench fp8 $sc rc=$?"
done
timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/bench_n2.log 2>&1; echo "bench n2 rc=$?"
FSDP_B200_CE=1 timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/bench_n2_ce.log 2>&1; echo "bench n2 ce rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["ms_per_step"], d["config"]["workload"][:48], (d.get("wire") or {}).get("GBps_per_direction"), d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
