# Round 2: fp8 push with the amax on the loaded words (40 registers): fp8 parity tests, the
# full-size W=8 emulated fp8 push, fp8 benches (delayed / dynamic), ncu of the fp8 push.
O=gpurun_out/${1:-r2fp8}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fp8_scaling.py tests/test_gpu_p2p.py tests/test_gpu_parity.py -q -x > $O/pytest_fp8.log 2>&1; echo "pytest fp8 rc=$?"; tail -2 $O/pytest_fp8.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -k "push" > $O/pytest_full.log 2>&1; echo "pytest full push rc=$?"; tail -2 $O/pytest_full.log
for sc in delayed dynamic; do
timeout 600 python bench.py --workload llama3.1-8b-fp8 --fp8-scaling $sc --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/bench_fp8_$sc.log 2>&1; echo "bench fp8 $sc rc=$?"
done
timeout 600 python bench.py --no-e2e --no-cpu-baseline --out $O/bench.jsonl > $O/bench_n1.log 2>&1; echo "bench n1 rc=$?"
B="python bench.py --workload llama3.1-8b-fp8 --fp8-scaling delayed --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:^k_" -c 600 --csv \
   --log-file $O/launches_fp8d.csv $B > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_unshard_push" -s 40 -c 1 -o $O/prof_fp8d_push $B > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python - <<PY
import json
for l in open("$O/bench.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["ms_per_step"], d["config"]["workload"][:60], d["isolated"]["ms_per_step"], {k: (v["avg_us"], v["GBps"]) for k, v in d["kernels_serial"].items()})
PY
