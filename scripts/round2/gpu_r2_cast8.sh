# The TMA cast for the fp8 W=1 unshard too (mixed e4m3 / bf16 tiles, fused amax): fp8 parity
# (scaling sequences, full-size W=1 block, fused amax), fp8 benches delayed / dynamic, bf16 bench
O=gpurun_out/${1:-r2cast8}
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_fp8_scaling.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_graphs.py tests/test_gpu_training_step.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for sc in delayed dynamic; do
  timeout 600 python bench.py --workload llama3.1-8b-fp8 --fp8-scaling $sc --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/b_fp8_$sc.log 2>&1; echo "fp8 $sc rc=$?"
done
timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/b_bf16.log 2>&1; echo "bf16 rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"][:60], d["ms_per_step"], d["ms_per_step_pct"]["median"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
