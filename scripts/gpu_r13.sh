# usage (under gpurun, 1 GPU): bash scripts/gpu_r13.sh TAG
TAG=${1:-r13}
mkdir -p gpurun_out
timeout 900 python scripts/stage_bench.py --no-torch --out gpurun_out/${TAG}_stages_8b.jsonl > gpurun_out/${TAG}_stages_8b.log 2>&1
echo "stage_bench rc=$?"
S="python scripts/stage_bench.py --ws 4 --iters 1 --warmup 0 --no-torch"
$S > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_rs_scatter|k_rs_pull_bulk" -c 3 \
    -o gpurun_out/${TAG}_prof_store_w4 $S > gpurun_out/${TAG}_ncu_store.log 2>&1
echo "ncu store rc=$?"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base \
    -k "regex:k_copy|k_rs|k_amax|k_fp8|k_unshard|k_pull|k_gather|k_signal|nccl" -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches_base.csv $B > gpurun_out/${TAG}_ncu_base.log 2>&1
echo "launch list (clock-control base) rc=$?"
