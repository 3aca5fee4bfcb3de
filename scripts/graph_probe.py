#!/usr/bin/env python3
"""Probe: can one toy FSDP step (unshard -> reshard -> reduce-scatter for every unit) be
captured into a CUDA graph through the library, and what does replay save over eager issue?
W=1 on one GPU, or under torchrun for W>1.  Prints one JSON line per rank 0."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
import paper_2410_06511_b200 as F  # noqa: E402


def main():
    W = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if W > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        mesh = F.Mesh.from_process_group(device=local)
    else:
        mesh = F.Mesh(1, 0, local, unique_id=F.get_unique_id())
    units = synth.model_units("toy")
    layers, grads = [], []
    for u in units:
        shapes = [s for _, s, _ in u]
        l = F.fsdp_shard(mesh, None, [e for _, _, e in u], shapes=shapes)
        l.sharded_flat().normal_(0, 0.02)
        layers.append(l)
        grads.append([torch.randn(s, device="cuda").to(torch.bfloat16) for s in shapes])
    s = torch.cuda.Stream()

    def step():
        F.fsdp_unshard(layers[0], stream=s)
        for i, l in enumerate(layers):
            F.fsdp_wait_unshard(l, stream=s)
            if i + 1 < len(layers):
                F.fsdp_unshard(layers[i + 1], stream=s)
            F.fsdp_reshard(l, stream=s)
            F.reduce_scatter_grads(l, grads[i], stream=s)
        for l in layers:
            F.fsdp_wait_reduce_scatter(l, stream=s)

    def timed(fn, n=200):
        torch.cuda.synchronize()
        if W > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(n):
            fn()
        e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1) / n * 1e3, (time.perf_counter() - t0) / n * 1e6

    with torch.cuda.stream(s):
        for _ in range(5):
            step()
    eager_dev_us, eager_host_us = timed(step)
    ref = [l.sharded_grad_flat().clone() for l in layers]
    out = {"W": W, "algo": mesh.algo if W > 1 else "local", "eager_us_per_step": round(eager_dev_us, 1),
           "eager_host_us_per_step": round(eager_host_us, 1)}
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        for l in layers:
            l.sharded_grad_flat().zero_()

        def replay():
            with torch.cuda.stream(s):   # replay() launches on the current stream
                g.replay()
        replay()
        torch.cuda.synchronize()
        same = all(torch.equal(l.sharded_grad_flat(), r) for l, r in zip(layers, ref))
        gdev, ghost = timed(replay)
        out.update({"graph": "captured", "replay_matches_eager": same, "graph_us_per_step": round(gdev, 1),
                    "graph_host_us_per_step": round(ghost, 1)})
    except Exception as e:   # noqa: BLE001 (probe: report whatever capture does)
        out.update({"graph": "failed", "error": f"{type(e).__name__}: {str(e).splitlines()[0][:300]}"})
    if rank == 0:
        print(json.dumps(out), flush=True)
    try:
        torch.cuda.synchronize()
        for l in layers:
            l.destroy()
        mesh.destroy()
    except Exception as e:   # noqa: BLE001
        if rank == 0:
            print(json.dumps({"teardown_error": str(e)[:200]}))
    if W > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
