# A/B: the TMA-load push at W > 1 (FSDP_B200_VARIANT=206 = 78 + 128) vs the register push (78):
# emulated push parity with bit 128, multi-GPU worker with it, benches N=2 / N=4 alternating
O=gpurun_out/${1:-r2tmapush}
mkdir -p $O
FSDP_B200_VARIANT=206 timeout 1200 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_fullsize.py tests/test_gpu_property.py -q -x -k "push or property" > $O/pytest_push.log 2>&1; echo "pytest push v206 rc=$?"; tail -1 $O/pytest_push.log
FSDP_B200_VARIANT=206 timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu v206 rc=$?"; tail -1 $O/pytest_mgpu.log
for i in 1 2; do for v in 78 206; do for n in 2 4; do
  FSDP_B200_VARIANT=$v timeout 600 python bench.py --gpus $n --no-e2e --no-cpu-baseline --out $O/v${v}_n$n.jsonl > $O/b_v${v}_n${n}_$i.log 2>&1; echo "v$v n$n rc=$?"
done; done; done
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d["ms_per_step"], d["ms_per_step_pct"]["median"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items() if k != "handshake"})
PY
