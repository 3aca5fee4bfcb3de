# A/B on one box: W=1 bf16 push with 2 (current) vs 3 (_ab_old/) smem output stages, alternating
O=gpurun_out/${1:-r2push3}
mkdir -p $O
for i in 1 2; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/s2.jsonl > $O/s2_$i.log 2>&1; echo "s2 rc=$?"
  (cd _ab_old && timeout 600 python bench.py --no-e2e --no-cpu-baseline --out ../$O/s3.jsonl > ../$O/s3_$i.log 2>&1); echo "s3 rc=$?"
done
(cd _ab_old && timeout 600 python -m pytest ../tests/test_gpu_parity.py -q -x -k "full_path_w1" > ../$O/pytest_s3.log 2>&1); echo "pytest s3 rc=$?"; tail -1 $O/pytest_s3.log
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d["ms_per_step"], d["ms_per_step_pct"]["median"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()}, d["roofline"]["frac"])
PY
