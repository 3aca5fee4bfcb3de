# A/B on one box: handshake with the single-thread system fences (default) vs without
# (-DFSDP_HS_NO_FENCE, _ab_old/), toy CUDA-graph step at N=2 and the 8B step at N=2
O=gpurun_out/${1:-r2fence}
mkdir -p $O
for i in 1 2; do
  (cd _ab_old && timeout 600 python bench.py --gpus 2 --workload toy --graph --steps 300 --warmup 30 --no-e2e --no-cpu-baseline --out ../$O/toy_nofence.jsonl > ../$O/t_nf_$i.log 2>&1); echo "nofence rc=$?"
  timeout 600 python bench.py --gpus 2 --workload toy --graph --steps 300 --warmup 30 --no-e2e --no-cpu-baseline --out $O/toy_fence.jsonl > $O/t_f_$i.log 2>&1; echo "fence rc=$?"
done
(cd _ab_old && timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out ../$O/b8_nofence.jsonl > ../$O/b_nf.log 2>&1); echo "8b nofence rc=$?"
timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out $O/b8_fence.jsonl > $O/b_f.log 2>&1; echo "8b fence rc=$?"
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d["n_gpus"], d["ms_per_step"], d["ms_per_step_pct"]["median"])
PY
