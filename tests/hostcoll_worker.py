"""Cross-process P2P parity on ONE GPU (host-collective mesh, no NCCL), launched by
tests/test_gpu_hostcoll.py:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port 29556 tests/hostcoll_worker.py

Every rank is its own process on cuda:0 (NCCL refuses two ranks on one GPU; CUDA IPC does
not), so the real multi-process P2P protocol runs where a one-GPU box can run it: symmetric
buffers exchanged as CUDA IPC handles and opened in every other process, the push unshard
and the pull / store reduce-scatter reading and writing the other processes' buffers, the
device-epoch ready/done handshakes between processes, the fp8 amax all-reduce over
symmetric memory, CUDA-graph replays, HSDP's world reduce-scatter and the handshake
timeout.  Only the link differs from a multi-GPU box (here the "peer" memory is local
HBM).  Host steps (IPC handle exchange, layout-hash check, barriers) go through
torch.distributed over gloo.  Every check is the multi-GPU worker's (tests/mgpu_worker.py)
against the oracle's World(W) / HsdpWorld simulation: bit-exact unshard (bf16 / e4m3),
bit-exact ascending-rank (FSDP) / nested-order (HSDP) fp32 reduce-scatter."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2410_06511_b200 as F  # noqa: E402
import mgpu_worker as M  # noqa: E402


def _device(rank):
    # every rank on cuda:0 by default; HOSTCOLL_SPREAD=1 puts rank r on GPU r % n (several
    # processes per GPU, peers both on the same GPU and across NVLink)
    if os.environ.get("HOSTCOLL_SPREAD") == "1":
        return rank % torch.cuda.device_count()
    return 0


def _hc_mesh(local, shard_size=None):
    return F.Mesh(dist.get_world_size(), dist.get_rank(), _device(dist.get_rank()), host_group=dist.group.WORLD,
                  shard_size=shard_size)


def main():
    rank = int(os.environ["RANK"])
    W = int(os.environ["WORLD_SIZE"])
    dev = _device(rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    mesh = _hc_mesh(dev)
    assert mesh.algo == "p2p" and mesh.hostcoll
    try:
        mesh.set_algo("nccl")
        raise AssertionError("set_algo(nccl) on a host-collective mesh must fail")
    except F.FsdpError as e:
        assert e.status_name == "FSDP_ERR_UNAVAILABLE", e
    for rs_mode in ("store", "pull"):
        mesh.set_p2p_rs(rs_mode)
        M.run_checks(mesh, W, rank, dev, "p2p")
        print(f"rank {rank}/{W} hostcoll rs={rs_mode}: unshard bf16/fp8 + reduce-scatter OK", flush=True)
    mesh.set_p2p_rs("auto")
    M.run_graph_checks(mesh, W, rank, "p2p")
    print(f"rank {rank}/{W} hostcoll: CUDA graph replays OK", flush=True)
    mesh.synchronize(120000)
    mesh.destroy()
    for Ws in sorted({d for d in (1, 2, W // 2) if 1 <= d < W and W % d == 0}):
        M.run_hsdp_checks(W, rank, dev, Ws, make_mesh=_hc_mesh)
    M.run_fault_injection(W, rank, dev, make_mesh=_hc_mesh)
    dist.barrier()
    dist.destroy_process_group()
    print(f"RANK {rank}/{W} hostcoll OK", flush=True)


if __name__ == "__main__":
    main()
