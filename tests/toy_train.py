"""A toy training loop through the library, compared with a single-device run — the
paper's correctness method ("We assume the correctness of FSDP, which can be further
verified by comparing it with DDP or even single-device jobs"; Table 7 /
Figure 4 compare loss curves against an FSDP ground truth).

Model: 2 residual MLP blocks (RMS-norm weight, w1 (768, 256), w2 (256, 768)), each block one
FSDP unit.  Mixed precision as in PAPER.md:417: bf16 all-gathered
parameters and compute, fp32 gradient reduce-scatter and fp32 master weights (SGD).

FSDP run (per rank r of W): unshard each block (bf16 views of library memory), forward on
the rank's micro-batch, backward into bf16 grads, reduce_scatter_grads (mean over ranks),
SGD on the fp32 shards.  Reference (single device): fp32 master params cast to bf16, the
same forward/backward on every rank's micro-batch, fp32 mean of the bf16 grads over ranks,
SGD on the fp32 masters.  Used by tests/test_gpu_training_step.py (W=1) and
tests/mgpu_worker.py (W = 2, 4)."""
import numpy as np
import torch

import synth

DIM, FFN = 256, 768


def block_shapes():
    return [(DIM,), (FFN, DIM), (DIM, FFN)]


def init_params(n_blocks=2):
    return [[synth.param_values(900 + b, p, s) for p, s in enumerate(block_shapes())] for b in range(n_blocks)]


def batch(step, rank, tokens=64):
    rng = np.random.default_rng(np.random.SeedSequence([241006511, 77, step, rank]))
    return torch.from_numpy(rng.standard_normal((tokens, DIM), dtype=np.float32)).cuda().to(torch.bfloat16)


def block_fwd(x, norm_w, w1, w2):
    h = x.float()
    h = (h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + 1e-6)).to(torch.bfloat16) * norm_w
    return x + torch.nn.functional.linear(torch.nn.functional.gelu(torch.nn.functional.linear(h, w1)), w2)


def loss_of(x, blocks):
    for p in blocks:
        x = block_fwd(x, *p)
    return x.float().pow(2).mean()


def reference_steps(n_steps, W, lr=0.05, n_blocks=2):
    """Single-device: returns the fp32 master params after each step."""
    master = [[torch.from_numpy(p).cuda() for p in blk] for blk in init_params(n_blocks)]
    # IEEE division by W ("a single division kernel"): a 0-dim CUDA divisor, because
    # torch divides by a CPU scalar as x * (1/W), which differs from x / W when W != 2^k
    div = torch.tensor(float(W), device="cuda")
    history = []
    for step in range(n_steps):
        grads = [[torch.zeros_like(p) for p in blk] for blk in master]
        for r in range(W):
            params = [[p.to(torch.bfloat16).requires_grad_() for p in blk] for blk in master]
            loss_of(batch(step, r), params).backward()
            for gb, pb in zip(grads, params):
                for g, p in zip(gb, pb):
                    g += p.grad.float() / div          # fp32 mean of the per-rank bf16 grads
        for mb, gb in zip(master, grads):
            for m, g in zip(mb, gb):
                m -= lr * g
        history.append([[m.clone() for m in blk] for blk in master])
    return history


def fsdp_steps(F, mesh, rank, n_steps, lr=0.05, n_blocks=2):
    """Through the library: returns this rank's fp32 shard views after each step (copied)."""
    layers = [F.fsdp_shard(mesh, [torch.from_numpy(p) for p in blk], [True, True, False])
              for blk in init_params(n_blocks)]
    history = []
    for step in range(n_steps):
        x = batch(step, rank)
        params = []
        F.fsdp_unshard(layers[0], torch.bfloat16)
        for i, l in enumerate(layers):                      # forward unshards with prefetch
            F.fsdp_wait_unshard(l)
            if i + 1 < len(layers):
                F.fsdp_unshard(layers[i + 1], torch.bfloat16)
            params.append([t.detach().requires_grad_() for t in l.unsharded_params()])
        loss_of(x, params).backward()
        for l, pb in zip(layers, params):
            F.reduce_scatter_grads(l, [p.grad for p in pb])  # fp32 reduce, mean over ranks
        for l in layers:
            F.fsdp_wait_reduce_scatter(l)
            F.fsdp_reshard(l)
            for p in range(l.P):                             # SGD on the fp32 shard
                shard = l.sharded_param(p)
                shard -= lr * l.sharded_grad(p)
        torch.cuda.synchronize()
        history.append([[l.sharded_param(p).clone() for p in range(l.P)] for l in layers])
    metas = [l.metas for l in layers]
    for l in layers:
        l.destroy()
    return history, metas


def compare(ref_hist, fsdp_hist, layers_meta, exact: bool):
    """Rank's shards vs the reference masters' rows. exact: bit-equality (W=1)."""
    for step, (ref, got) in enumerate(zip(ref_hist, fsdp_hist)):
        for b, (rblk, gblk) in enumerate(zip(ref, got)):
            for p, (rm, gs) in enumerate(zip(rblk, gblk)):
                m = layers_meta[b][p]
                rows = rm.reshape(m["dim0"], -1)[m["row_begin"]:m["row_begin"] + m["row_count"]].reshape(gs.shape)
                if exact:
                    assert torch.equal(rows, gs), (step, b, p)
                else:
                    torch.testing.assert_close(gs, rows, rtol=1e-5, atol=1e-6)
