# final multi-GPU confirmation of the final code: multi-GPU worker (W=4 and 2), default bench N=4 and N=2
O=gpurun_out/${1:-r2mgfinal}
mkdir -p $O
timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "pytest mgpu rc=$?"; tail -1 $O/pytest_mgpu.log
for n in 4 2; do
  timeout 900 python bench.py --gpus $n --out $O/bench.jsonl > $O/b_n$n.log 2>&1; echo "bench n$n rc=$?"; grep '^{' $O/b_n$n.log | cut -c1-200
done
