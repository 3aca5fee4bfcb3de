# Round 2: handshakes fenced only where the protocol publishes unfenced local writes: the
# multi-GPU worker 3x (W=4 and W=2 each), the one-GPU multi-process tests, toy graph and 8B
# steps at N=2 / N=4 (under gpurun --gpus 4)
O=gpurun_out/${1:-r2fence2}
mkdir -p $O
for i in 1 2 3; do
  timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu_$i.log 2>&1; echo "pytest mgpu run $i rc=$?"; tail -1 $O/pytest_mgpu_$i.log
done
timeout 900 python -m pytest tests/test_gpu_hostcoll.py tests/test_gpu_graphs.py -q -x > $O/pytest_hc.log 2>&1; echo "pytest hostcoll rc=$?"; tail -1 $O/pytest_hc.log
B="python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl"
for n in 2 4; do
  timeout 600 $B --gpus $n --workload toy --graph --steps 300 --warmup 30 > $O/toy_n$n.log 2>&1; echo "toy n$n rc=$?"
  timeout 600 $B --gpus $n > $O/b_n$n.log 2>&1; echo "8b n$n rc=$?"
done
timeout 600 $B --gpus 4 --shard-size 2 > $O/b_hsdp.log 2>&1; echo "hsdp rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["config"]["shard_size"], d["config"]["workload"][:12], d["ms_per_step"], d["ms_per_step_pct"]["median"])
PY
