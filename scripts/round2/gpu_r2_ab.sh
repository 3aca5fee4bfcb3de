# Round 2 A/B on one box: K5 TMA stages 2 vs 4 at N=1 (twice each), N=2 twice
O=gpurun_out/${1:-r2ab}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rs_copy_in or full" > $O/pytest_k5.log 2>&1; echo "pytest k5 rc=$?"; tail -1 $O/pytest_k5.log
FSDP_B200_K5_STAGES=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "rs_copy_in or w1" > $O/pytest_k5s4.log 2>&1; echo "pytest k5 stages4 rc=$?"; tail -1 $O/pytest_k5s4.log
for i in 1 2; do
  for st in 2 4; do
    FSDP_B200_K5_STAGES=$st timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/bench_k5s$st.jsonl > $O/b_n1_s${st}_$i.log 2>&1; echo "n1 k5 stages $st rc=$?"
  done
  timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out $O/bench_n2.jsonl > $O/b_n2_$i.log 2>&1; echo "n2 rc=$?"
done
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/bench*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d["n_gpus"], d["ms_per_step"], d["ms_per_step_pct"]["median"], d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()}, d["roofline"]["frac"], d["roofline"].get("step_hbm_frac"))
PY
