# usage: bash scripts/gpu_profile.sh TAG — bench + ncu launch list + ncu --set full of the W=1 kernels
TAG=${1:-r07}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:k_copy|k_rs|k_amax|k_fp8|k_unshard|k_pull|k_gather|k_signal|nccl" -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_list.log 2>&1
echo "launch list rc=$?"
$B > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_unshard_push|k_rs_copy_in" -s 2 -c 2 \
    -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
