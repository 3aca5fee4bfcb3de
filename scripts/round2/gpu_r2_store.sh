# Round 2: full-size parity + own-row store RS + NVLink wire bytes (under gpurun --gpus 2)
O=gpurun_out/r2s
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_p2p.py -q -x --durations=10 > $O/pytest_new.log 2>&1; echo "pytest new rc=$?"; tail -3 $O/pytest_new.log
timeout 900 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -2 $O/pytest_mgpu.log
for rs in auto store pull; do
  timeout 600 python bench.py --gpus 2 --p2p-rs $rs --grads library --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_n2_$rs.log 2>&1; echo "bench n2 $rs rc=$?"
done
FSDP_B200_STORE_OWN=0 timeout 600 python bench.py --gpus 2 --p2p-rs store --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_n2_store_noown.log 2>&1; echo "bench n2 store noown rc=$?"
timeout 600 python bench.py --gpus 2 --p2p-rs store --grads torch --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_n2_store_torch.log 2>&1; echo "bench n2 store torch rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r2s/bench.jsonl"):
    d = json.loads(l)
    print(d["ms_per_step"], d["config"]["collectives"], d["config"]["grads"], d.get("wire", {}) and d["wire"]["GBps_per_direction"], d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
timeout 300 python scripts/nvlink_wire.py --W 2 > $O/wire_w2.jsonl 2>&1; echo "wire rc=$?"; cat $O/wire_w2.jsonl | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"k_unshard_push|k_rs_pull|k_rs_scatter" --csv --log-file $O/ncu_wire_w2.csv python scripts/nvlink_wire.py --W 2 --iters 1 > $O/ncu_wire.log 2>&1; echo "ncu wire rc=$?"; tail -3 $O/ncu_wire.log
