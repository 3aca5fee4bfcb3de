mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 17 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_p2p.py -q -x \
  -k "(ragged-1 or ragged-4 or toyroot) and not exhaustive and not all_fp32 and not llama8b and not prefetch and not state" \
  > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid|out of bounds" gpurun_out/memcheck.log | head -20
