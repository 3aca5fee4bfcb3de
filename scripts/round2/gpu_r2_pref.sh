# Round 2: bf16 push with a register double buffer (bf16-only kernel, 31 registers):
# push parity (emulated W, full size), benches N=1 (x2) and N=2
O=gpurun_out/${1:-r2pref}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_parity.py tests/test_gpu_property.py -q -x > $O/pytest_push.log 2>&1; echo "pytest push rc=$?"; tail -2 $O/pytest_push.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x > $O/pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -2 $O/pytest_full.log
for i in 1 2; do timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/b_n1_$i.log 2>&1; echo "n1 rc=$?"; done
FSDP_B200_CTAS_PER_SM=8 timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/bench_cta8.jsonl > $O/b_n1_cta8.log 2>&1; echo "n1 cta8 rc=$?"
timeout 600 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/b_n2.log 2>&1; echo "n2 rc=$?"
python - <<PY
import json
for f in ["$O/bench.jsonl", "$O/bench_cta8.jsonl"]:
    for l in open(f):
        d = json.loads(l)
        print(f[-12:], d["n_gpus"], d["ms_per_step"], d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()}, d["roofline"]["frac"], d["roofline"].get("step_hbm_frac"))
PY
