# Round 2: copy-engine transfer path (FSDP_B200_CE=1) on 4 GPUs: emulated parity of the CE
# offsets, the CE wire probe, multi-GPU parity, benches N=2/4 with and without CE
O=gpurun_out/r2ce
mkdir -p $O
FSDP_B200_CE=1 timeout 1500 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_fullsize.py -q -x -k "push or store or w8" > $O/pytest_ce_emul.log 2>&1; echo "pytest ce emul rc=$?"; tail -2 $O/pytest_ce_emul.log
for w in 2 4; do timeout 300 python scripts/nvlink_wire.py --W $w --kernels push,ce > $O/wire_ce_w$w.jsonl 2>&1; echo "wire ce w$w rc=$?"; cut -c1-160 $O/wire_ce_w$w.jsonl; done
FSDP_B200_CE=1 timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu_ce.log 2>&1; echo "pytest mgpu ce rc=$?"; tail -2 $O/pytest_mgpu_ce.log
for n in 2 4; do
  for ce in 0 1; do
    FSDP_B200_CE=$ce timeout 600 python bench.py --gpus $n --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_n${n}_ce$ce.log 2>&1; echo "bench n$n ce$ce rc=$?"
  done
  FSDP_B200_CE=1 timeout 600 python bench.py --gpus $n --workload llama3.1-8b-fp8 --fp8-scaling delayed --no-cpu-baseline --no-e2e --out $O/bench.jsonl > $O/bench_fp8_n${n}_ce1.log 2>&1; echo "bench fp8 n$n ce1 rc=$?"
done
python - <<'PY'
import json
for l in open("gpurun_out/r2ce/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["ms_per_step"], d["config"]["workload"][:40], d["config"]["collectives"], (d.get("wire") or {}).get("GBps_per_direction"), d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
