#!/usr/bin/env python3
"""Unshard/reshard message-size sweep (BASELINE.json configs[4]): 64 KB - 1 GB of bf16
all-gather output per unit, ragged per-parameter shapes (synth.sweep_unit: d0 not divisible
by W, a param with d0 < W, odd `rest`), at W = 2/4/8 GPUs, for the fused P2P path and the
NCCL path, next to plain NCCL all-gather / reduce-scatter of contiguous buffers of the
same sizes (the NCCL ceiling, torch.distributed).  One JSON line per (size, variant).

    torchrun --nproc-per-node W scripts/sweep_bench.py [--iters 20] [--out file]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
import paper_2410_06511_b200 as F  # noqa: E402


def fit_alpha_B(lines, W):
    """Least-squares fit of the alpha-beta cost model t = alpha + x / B per variant and
    collective (SPEC.md:673's latency + bytes/bandwidth model), x = bus bytes
    (W-1)/W * algorithm bytes; alpha in us, B in GB/s."""
    import numpy as np
    out = []
    for var in sorted({l["variant"] for l in lines}):
        rows = [l for l in lines if l["variant"] == var]
        for op, key, mult in (("unshard", "unshard_us", 1), ("reduce_scatter", "rs_us", 2)):
            x = np.array([l["ag_bytes"] * mult * (W - 1) / W for l in rows], dtype=np.float64)
            t = np.array([l[key] for l in rows], dtype=np.float64)
            if len(x) < 2 or W == 1:
                continue
            A = np.stack([np.ones_like(x), x], axis=1) / t[:, None]     # relative residuals:
            (alpha, inv_b), *_ = np.linalg.lstsq(A, np.ones_like(t), rcond=None)  # small sizes count
            out.append({"fit": "alpha_B", "variant": var, "op": op, "W": W, "points": len(x),
                        "alpha_us": round(float(alpha), 2),
                        "B_GBps": round(float(1e-3 / inv_b), 1) if inv_b > 0 else None})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--min-log2", type=int, default=16)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--out", default=None)
    ap.add_argument("--graph", action="store_true",
                    help="time CUDA-graph replays of each library op (captured once after the warm-up): the "
                         "device-side latency alpha without host launch overhead; the NCCL ceiling stays eager")
    args = ap.parse_args()
    W = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    mesh = F.Mesh.from_process_group(device=local)
    comp = torch.cuda.Stream(device=dev)
    lines = []
    algos = ["p2p", "nccl"] if mesh.algo == "p2p" else ["nccl"]

    def timed(fn, graph=False):
        for _ in range(3):
            fn()
        comp.synchronize()
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=comp):
                fn()

            def fn():   # noqa: F811 (replays on the capture stream)
                with torch.cuda.stream(comp):
                    g.replay()
            fn()
            comp.synchronize()
        dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        for _ in range(args.iters):
            fn()
        e1.record(comp)
        comp.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.iters], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for lg in range(args.min_log2, args.max_log2 + 1):
        T = 1 << lg
        unit = synth.sweep_unit(T, W)
        shapes = [s for _, s, _ in unit]
        for algo in algos:
            mesh.set_algo(algo)
            layer = F.fsdp_shard(mesh, None, [False] * len(shapes), shapes=shapes)
            layer.sharded_flat().normal_(0, 0.02)
            grads = layer.full_grad_buffers(torch.bfloat16) if algo == "p2p" else \
                [torch.randn(s, device=dev).to(torch.bfloat16) for s in shapes]
            for g in grads:
                g.normal_(0, 1e-3)

            def unshard():
                F.fsdp_unshard(layer, torch.bfloat16, stream=comp)
                F.fsdp_wait_unshard(layer, stream=comp)
                F.fsdp_reshard(layer, stream=comp)

            def rs():
                F.reduce_scatter_grads(layer, grads, stream=comp)
                F.fsdp_wait_reduce_scatter(layer, stream=comp)

            ms_u = timed(unshard, args.graph)
            ms_r = timed(rs, args.graph)
            ag_bytes = W * 2 * layer.S
            rs_bytes = W * 4 * layer.S
            busbw = (ag_bytes + rs_bytes) * (W - 1) / W / ((ms_u + ms_r) * 1e-3) / 1e9
            lines.append({"log2_bytes": lg, "variant": f"fsdp_{algo}" + ("_graph" if args.graph else ""), "W": W,
                          "params": len(shapes),
                          "ag_bytes": ag_bytes, "unshard_us": round(ms_u * 1e3, 2), "rs_us": round(ms_r * 1e3, 2),
                          "unshard_busbw_GBps": round(ag_bytes * (W - 1) / W / (ms_u * 1e-3) / 1e9, 1),
                          "rs_busbw_GBps": round(rs_bytes * (W - 1) / W / (ms_r * 1e-3) / 1e9, 1),
                          "busbw_GBps": round(busbw, 1), "frac_900": round(busbw / 900, 4)})
            layer.destroy()
        # NCCL ceiling: contiguous all-gather (T bytes bf16 out) and reduce-scatter (2T bytes fp32 in)
        n = max(W, (T // 2) // W * W)
        ag_out = torch.empty(n, dtype=torch.bfloat16, device=dev)
        ag_in = torch.randn(n // W, device=dev).to(torch.bfloat16)
        rs_in = torch.randn(n, dtype=torch.float32, device=dev)
        rs_out = torch.empty(n // W, dtype=torch.float32, device=dev)

        def nccl_ag():
            with torch.cuda.stream(comp):
                dist.all_gather_into_tensor(ag_out, ag_in)

        def nccl_rs():
            with torch.cuda.stream(comp):
                dist.reduce_scatter_tensor(rs_out, rs_in)

        ms_a = timed(nccl_ag)
        ms_b = timed(nccl_rs)
        busbw = (2 * n + 4 * n) * (W - 1) / W / ((ms_a + ms_b) * 1e-3) / 1e9
        lines.append({"log2_bytes": lg, "variant": "nccl_contiguous_ceiling", "W": W, "ag_bytes": 2 * n,
                      "unshard_us": round(ms_a * 1e3, 2), "rs_us": round(ms_b * 1e3, 2),
                      "busbw_GBps": round(busbw, 1), "frac_900": round(busbw / 900, 4)})
        if rank == 0:
            for l in lines[-3:]:
                print(json.dumps(l), flush=True)
    if rank == 0:
        fits = fit_alpha_B(lines, W)
        for l in fits:
            print(json.dumps(l), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                for l in lines + fits:
                    f.write(json.dumps(l) + "\n")
    mesh.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
