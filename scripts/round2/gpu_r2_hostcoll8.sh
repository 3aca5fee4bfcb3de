# Round 2: host-collective mesh at W = 8: 8 processes on one GPU, then 8 processes spread
# over the visible GPUs (rank r on GPU r % n: peers on the same GPU and across NVLink)
O=gpurun_out/${1:-r2hc8}
mkdir -p $O
P=$(python -c "import socket;s=socket.socket();s.bind(('127.0.0.1',0));print(s.getsockname()[1])")
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 \
  --master-port $P tests/hostcoll_worker.py > $O/hostcoll_n8.log 2>&1; echo "hostcoll n8 one GPU rc=$?"; grep -o "hostcoll OK" $O/hostcoll_n8.log | wc -l
P=$(python -c "import socket;s=socket.socket();s.bind(('127.0.0.1',0));print(s.getsockname()[1])")
HOSTCOLL_SPREAD=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 \
  --master-port $P tests/hostcoll_worker.py > $O/hostcoll_n8_spread.log 2>&1; echo "hostcoll n8 spread rc=$?"; grep -o "hostcoll OK" $O/hostcoll_n8_spread.log | wc -l
grep "rank 0/8" $O/hostcoll_n8.log | cut -c1-200
