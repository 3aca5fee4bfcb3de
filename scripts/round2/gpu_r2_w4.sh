# Round 2 on 4 GPUs: CE schedules probe, NVLink wire bytes at W=4, fp8 delayed (fused amax)
# tests + benches, multi-GPU parity at W=2/4, bench N=4 variants (under gpurun --gpus 4)
O=gpurun_out/r2w4
mkdir -p $O
timeout 300 python scripts/ce_probe.py --W 2 > $O/ce_w2.jsonl 2>&1; echo "ce w2 rc=$?"; cat $O/ce_w2.jsonl
timeout 300 python scripts/ce_probe.py --W 4 > $O/ce_w4.jsonl 2>&1; echo "ce w4 rc=$?"; cat $O/ce_w4.jsonl
timeout 900 python -m pytest tests/test_gpu_fp8_scaling.py tests/test_gpu_parity.py -q -x -k "fp8" > $O/pytest_fp8.log 2>&1; echo "pytest fp8 rc=$?"; tail -2 $O/pytest_fp8.log
timeout 300 python scripts/nvlink_wire.py --W 4 > $O/wire_w4.jsonl 2>&1; echo "wire w4 rc=$?"; cut -c1-200 $O/wire_w4.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"k_unshard_push|k_rs_pull|k_rs_scatter" --csv --log-file $O/ncu_wire_w4.csv python scripts/nvlink_wire.py --W 4 --iters 1 > $O/ncu_wire.log 2>&1; echo "ncu wire rc=$?"
timeout 1200 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -2 $O/pytest_mgpu.log
for n in 1 4; do
  timeout 600 python bench.py --gpus $n --workload llama3.1-8b-fp8 --fp8-scaling delayed --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_fp8d_n$n.log 2>&1; echo "bench fp8 delayed n$n rc=$?"
  timeout 600 python bench.py --gpus $n --workload llama3.1-8b-fp8 --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_fp8_n$n.log 2>&1; echo "bench fp8 dynamic n$n rc=$?"
done
timeout 900 python bench.py --gpus 4 --out $O/bench.jsonl > $O/bench_n4.log 2>&1; echo "bench n4 rc=$?"
for rs in store pull; do
  timeout 600 python bench.py --gpus 4 --p2p-rs $rs --grads library --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_n4_$rs.log 2>&1; echo "bench n4 $rs rc=$?"
done
python - <<'PY'
import json
for l in open("gpurun_out/r2w4/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["ms_per_step"], d["config"]["workload"][:60], d["config"]["collectives"], (d.get("wire") or {}).get("GBps_per_direction"), d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
