# HSDP 2x2 / 4x1: replica-gather grid (CTAs per SM 0 = default, 1, 2), twice each
O=gpurun_out/${1:-r2gather}
mkdir -p $O
for i in 1 2; do
  for g in 0 1 2; do
    FSDP_B200_GATHER_CTAS_PER_SM=$g timeout 600 python bench.py --gpus 4 --shard-size 2 --no-e2e --no-cpu-baseline --out $O/hsdp22_g$g.jsonl > $O/h22_g${g}_$i.log 2>&1; echo "2x2 g$g rc=$?"
  done
done
for g in 0 2; do
  FSDP_B200_GATHER_CTAS_PER_SM=$g timeout 600 python bench.py --gpus 4 --shard-size 1 --no-e2e --no-cpu-baseline --out $O/hsdp41_g$g.jsonl > $O/h41_g$g.log 2>&1; echo "4x1 g$g rc=$?"
done
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d["ms_per_step"], d["ms_per_step_pct"]["median"], d["ms_per_step_pct"]["p10"], d["ms_per_step_pct"]["p90"])
PY
