# K5 with 3 TMA stages as the default: W=1-path parity (every dtype combination), benches N=1 x2
O=gpurun_out/${1:-r2k5b}
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fp8_scaling.py tests/test_gpu_training_step.py tests/test_gpu_graphs.py tests/test_gpu_guards.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for i in 1 2; do timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/b_$i.log 2>&1; echo "n1 rc=$?"; done
timeout 600 python bench.py --workload llama3.1-8b-fp8 --fp8-scaling delayed --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/b_fp8.log 2>&1; echo "fp8 rc=$?"
timeout 600 python bench.py --workload llama3.1-70b --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/b_70b.log 2>&1; echo "70b rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"][:16], d["ms_per_step"], d["ms_per_step_pct"]["median"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()}, d["roofline"]["kernel"], d["roofline"]["frac"], d["roofline"]["step_hbm_frac"])
PY
