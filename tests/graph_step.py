"""A toy FSDP step through the library, written so that it can be captured into a CUDA graph
(shared by tests/test_gpu_graphs.py and tests/mgpu_worker.py): every unit is unsharded with
the next one prefetched, its params are consumed by a copy (the "forward"),
resharded, and its grads reduce-scattered; optionally the fp8 scales are precomputed first."""
import numpy as np
import torch

import synth


def setup(F, mesh, rank=0, seed=300):
    units = synth.model_units("toy")
    layers, grads, params = [], [], []
    for ui, u in enumerate(units):
        shapes = [s for _, s, _ in u]
        elig = [e for _, _, e in u]
        P = [synth.param_values(seed + ui, p, s) for p, s in enumerate(shapes)]
        params.append((shapes, elig, P))
        layers.append(F.fsdp_shard(mesh, [torch.from_numpy(x) for x in P], elig))
        grads.append([torch.from_numpy(synth.grad_bf16_bits(ui, p, rank, s).view(np.int16)).cuda().view(torch.bfloat16)
                      for p, s in enumerate(shapes)])
    return layers, grads, params


def outs_for(layers, fp8):
    res = []
    for l in layers:
        row = []
        for p, shp in enumerate(l.shapes):
            e = fp8 and l.fp8_eligible[p]
            row.append(torch.empty(shp, dtype=torch.uint8 if e else torch.bfloat16, device="cuda"))
        res.append(row)
    return res


def step(F, mesh, layers, grads, s, outs, fp8=False):
    dt = torch.float8_e4m3fn if fp8 else torch.bfloat16
    if fp8:
        F.precompute_fp8_scales(mesh, layers, stream=s)
    F.fsdp_unshard(layers[0], dt, stream=s)
    for i, l in enumerate(layers):
        F.fsdp_wait_unshard(l, stream=s)
        if i + 1 < len(layers):
            F.fsdp_unshard(layers[i + 1], dt, stream=s)
        for o, t in zip(outs[i], l.unsharded_params()):
            o.copy_(t.view(torch.uint8) if t.dtype == torch.float8_e4m3fn else t)
        F.fsdp_reshard(l, stream=s)
        F.reduce_scatter_grads(l, grads[i], stream=s)
    for l in layers:
        F.fsdp_wait_reduce_scatter(l, stream=s)


def refill(layers, grads, params, rank, seed):
    """New values written in place into the shards (this rank's rows of fresh params) and the
    grads; returns the new full params per unit."""
    for ui, l in enumerate(layers):
        shapes, elig, _ = params[ui]
        P2 = [synth.param_values(seed + ui, p, sh) for p, sh in enumerate(shapes)]
        for p in range(l.P):
            m = l.metas[p]
            rows = P2[p].reshape(m["dim0"], -1)[m["row_begin"]:m["row_begin"] + m["row_count"]]
            if rows.size:
                l.sharded_param(p).copy_(torch.from_numpy(np.ascontiguousarray(rows)).reshape(l.sharded_param(p).shape))
        params[ui] = (shapes, elig, P2)
        for p, sh in enumerate(shapes):
            grads[ui][p].copy_(torch.from_numpy(synth.grad_bf16_bits(ui + seed, p, rank, sh).view(np.int16))
                               .view(torch.bfloat16).reshape(sh))
    return params
