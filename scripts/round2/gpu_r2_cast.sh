# A/B: W=1 bf16 unshard as the TMA-in/TMA-out cast (FSDP_B200_VARIANT=78) vs the push (14)
O=gpurun_out/${1:-r2cast}
mkdir -p $O
FSDP_B200_VARIANT=78 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "full_path_w1 or w1_block or w1_root or unshard_bf16" > $O/pytest_v78.log 2>&1; echo "pytest v78 rc=$?"; tail -1 $O/pytest_v78.log
for i in 1 2; do for v in 14 78; do
  FSDP_B200_VARIANT=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/v$v.jsonl > $O/b_v${v}_$i.log 2>&1; echo "v$v rc=$?"
done; done
FSDP_B200_VARIANT=78 timeout 600 python bench.py --workload llama3.1-70b --no-e2e --no-cpu-baseline --out $O/v78_70b.jsonl > $O/b_70b.log 2>&1; echo "70b v78 rc=$?"
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d["ms_per_step"], d["ms_per_step_pct"]["median"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()}, d["roofline"]["kernel"], d["roofline"]["frac"])
PY
