# A/B on one box at N=2: the r2final library (b827882, _ab_old/) vs the current one, twice each
O=gpurun_out/${1:-r2ab2}
mkdir -p $O
for i in 1 2; do
  (cd _ab_old && timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out ../$O/bench_old.jsonl > ../$O/b_old_$i.log 2>&1); echo "old rc=$?"
  timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out $O/bench_new.jsonl > $O/b_new_$i.log 2>&1; echo "new rc=$?"
done
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/bench*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d["n_gpus"], d["ms_per_step"], d["ms_per_step_pct"]["median"], d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
