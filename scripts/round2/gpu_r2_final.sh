# Round 2 validation on the box's GPUs (1 or 4): smoke, every -m gpu test (multi-GPU worker at W=4 and W=2),
# default benches N=1/2/4 (e2e + CPU baseline), the reference arm at N=1, the ncu launch list
# of the N=1 bench and one ncu --set full capture of the W=1 kernels (under gpurun --gpus 4)
O=gpurun_out/${1:-r2final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpus.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2700 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
NG=$(nvidia-smi -L | wc -l)
for n in 1 2 4; do
  [ $n -gt $NG ] && continue
  timeout 900 python bench.py --gpus $n --out $O/bench.jsonl > $O/bench_n$n.log 2>&1; echo "bench n$n rc=$?"; grep '^{' $O/bench_n$n.log | cut -c1-240
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref rc=$?"; grep '^{' $O/bench_ref.log | cut -c1-240
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" -c 600 --csv \
   --log-file $O/launches_w1.csv $B > $O/ncu_launches.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_cast_w1|k_unshard_push|k_rs_copy_in" -s 40 -c 2 \
   -o $O/prof_w1 $B > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
