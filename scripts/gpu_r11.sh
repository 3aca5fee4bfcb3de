# usage (under gpurun, 1 GPU): bash scripts/gpu_r11.sh TAG
TAG=${1:-r11}
mkdir -p gpurun_out
bash scripts/gpu_all.sh
for f in smoke.log pytest_gpu.log bench_n1.log; do cp gpurun_out/$f gpurun_out/${TAG}_$f; done
bash scripts/gpu_profile.sh $TAG
S="python scripts/stage_bench.py --ws 4 --iters 1 --warmup 1 --no-torch"
$S > gpurun_out/${TAG}_stage_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_rs_pull_bulk|k_unshard_push_bulk" -c 2 \
    -o gpurun_out/${TAG}_prof_pull_w4 $S > gpurun_out/${TAG}_ncu_pull.log 2>&1
echo "ncu pull/push w4-emulated rc=$?"
