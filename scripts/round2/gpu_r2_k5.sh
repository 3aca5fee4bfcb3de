# K5 TMA stages 2 vs 3 at N=1 (alternating, twice each) + K5 parity with 3 stages
O=gpurun_out/${1:-r2k5}
mkdir -p $O
FSDP_B200_K5_STAGES=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "rs_copy_in or w1" > $O/pytest_k5s3.log 2>&1; echo "pytest k5 s3 rc=$?"; tail -1 $O/pytest_k5s3.log
for i in 1 2; do for st in 2 3; do
  FSDP_B200_K5_STAGES=$st timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/k5s$st.jsonl > $O/b_s${st}_$i.log 2>&1; echo "n1 s$st rc=$?"
done; done
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d["ms_per_step"], d["ms_per_step_pct"]["median"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()}, d["roofline"]["frac"])
PY
