# Round 2: HSDP two-phase world reduce-scatter (pieces + replica gather) vs the one-phase
# world pull: one-GPU emulated parity, multi-GPU worker (W=4 then W=2), benches 2x2 and 4x1
# (under gpurun --gpus 4)
O=gpurun_out/${1:-r2hsdp2}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_hsdp.py -q -x > $O/pytest_hsdp.log 2>&1; echo "pytest hsdp rc=$?"; tail -2 $O/pytest_hsdp.log
timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -2 $O/pytest_mgpu.log
for ss in 2 1; do
  timeout 600 python bench.py --gpus 4 --shard-size $ss --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_hsdp_s${ss}_2ph.log 2>&1; echo "bench hsdp shard $ss two-phase rc=$?"
  FSDP_B200_HSDP_RS=1 timeout 600 python bench.py --gpus 4 --shard-size $ss --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_hsdp_s${ss}_1ph.log 2>&1; echo "bench hsdp shard $ss one-phase rc=$?"
done
timeout 600 python bench.py --gpus 4 --shard-size 2 --step train --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_hsdp_train.log 2>&1; echo "bench hsdp 2x2 train rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["config"]["shard_size"], d["ms_per_step"], d["config"]["collectives"][-60:], (d.get("wire") or {}).get("GBps_per_direction"), d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
