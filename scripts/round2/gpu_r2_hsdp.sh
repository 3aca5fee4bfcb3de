# Round 2: HSDP world pull (one NVSwitch domain): one-GPU emulated parity, multi-GPU worker
# (W=4: HSDP 4x1 and 2x2, world pull bit-exact to the nested oracle order; then W=2), benches
# 2x2 world pull vs the NCCL pair vs FSDP-4 (under gpurun --gpus 4)
O=gpurun_out/${1:-r2hsdp}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_hsdp.py -q -x > $O/pytest_hsdp.log 2>&1; echo "pytest hsdp rc=$?"; tail -2 $O/pytest_hsdp.log
timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -2 $O/pytest_mgpu.log
timeout 600 python bench.py --gpus 4 --shard-size 2 --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_hsdp22_wp.log 2>&1; echo "bench hsdp 2x2 world pull rc=$?"
FSDP_B200_HSDP_P2P=0 timeout 600 python bench.py --gpus 4 --shard-size 2 --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_hsdp22_nccl.log 2>&1; echo "bench hsdp 2x2 nccl pair rc=$?"
timeout 600 python bench.py --gpus 4 --shard-size 1 --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_hsdp41_wp.log 2>&1; echo "bench hsdp 4x1 world pull rc=$?"
timeout 600 python bench.py --gpus 4 --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_fsdp4.log 2>&1; echo "bench fsdp4 rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["config"]["shard_size"], d["ms_per_step"], d["config"]["collectives"][:110], (d.get("wire") or {}).get("GBps_per_direction"), d["isolated"]["ms_per_step"])
PY
