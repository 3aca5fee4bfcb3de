"""Property suite over 1000 random uneven units (SPEC.md:807 acceptance #7: ">= 1000-case
property suite with uneven shapes"), the CUDA path against the oracle, bit for bit.

Each case draws (seeded) a world size W in [1, 8] and a unit of 1-6 params with 1-3 dims,
dim 0 in [0, 3W + 5] (so d0 = 0, d0 < W, d0 not divisible by W all occur), odd trailing
dims, random fp8 eligibility; then, with W communicator-less meshes on cuda:0, it checks
* every rank's fp32 shard (R1 layout, zero padding);
* the fused unshard (push kernel into W sentinel-filled arenas, bf16 or e4m3 with the
  oracle's scale): every arena holds cast(P_p) at the published offsets, nothing else written;
* the reduce-scatter (store-scatter + receive-reduce, or the pull, alternating): every rank's
  fp32 grad rows equal the oracle's ascending-rank sum of fp32(g_q) / W."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F

import synth  # noqa: E402
from oracle import World  # noqa: E402
from oracle.world import BF16, FP8  # noqa: E402

N_CASES = 1000
BATCH = 100
_MESHES = {}


def _mesh(W, r):
    if (W, r) not in _MESHES:
        _MESHES[(W, r)] = F.Mesh(W, r, 0, local=True)
    return _MESHES[(W, r)]


@pytest.fixture(scope="module", autouse=True)
def _cleanup():
    yield
    for m in _MESHES.values():
        m.destroy()
    _MESHES.clear()


def _case(i):
    rng = np.random.default_rng(np.random.SeedSequence([241006511, 807, i]))
    W = int(rng.integers(1, 9))
    shapes, elig = [], []
    for _ in range(int(rng.integers(1, 7))):
        d0 = int(rng.integers(0, 3 * W + 6))
        nd = int(rng.integers(1, 4))
        rest = tuple(int(x) for x in rng.choice([1, 3, 5, 7, 16, 17, 33], size=nd - 1))
        shapes.append((d0,) + rest)
        elig.append(bool(rng.integers(0, 2)) and nd == 2)
    return W, shapes, elig, rng


@pytest.mark.parametrize("batch", range(N_CASES // BATCH))
def test_property_batch(batch):
    for i in range(batch * BATCH, (batch + 1) * BATCH):
        W, shapes, elig, rng = _case(i)
        P = [synth.param_values(i, p, s) for p, s in enumerate(shapes)]
        w = World(shapes, W, elig)
        shards = w.shard(P)
        layers = [F.fsdp_shard(_mesh(W, r), [torch.from_numpy(x) for x in P], elig) for r in range(W)]
        try:
            for r, l in enumerate(layers):
                np.testing.assert_array_equal(l.sharded_flat().cpu().numpy().view(np.uint32),
                                              shards[r].view(np.uint32), err_msg=f"case {i} shard r={r}")
            # fused unshard
            fp8 = bool(i % 3 == 1) and any(elig)
            dt = torch.float8_e4m3fn if fp8 else torch.bfloat16
            scale = w.precompute_fp8_scales(shards)[1] if fp8 else None
            offs, total = F.unsharded_layout(layers[0], dt)
            arenas = [torch.full((total + 16,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(W)]
            sdev = torch.from_numpy(scale).cuda() if fp8 else None
            for l in layers:
                F.stage_unshard_push(l, dt, arenas, fp8_scales=sdev)
            _, fulls = w.unshard(shards, FP8 if fp8 else BF16, scale)
            for d in range(W):
                a = arenas[d].cpu().numpy()
                written = np.zeros(a.size, dtype=bool)
                for p, want in enumerate(fulls):
                    nb = want.size * want.itemsize
                    np.testing.assert_array_equal(a[offs[p]:offs[p] + nb].view(want.dtype).reshape(want.shape), want,
                                                  err_msg=f"case {i} unshard arena {d} param {p}")
                    written[offs[p]:offs[p] + nb] = True
                assert np.all(a[~written] == 0xA5), f"case {i}: unshard wrote outside the tensors"
            # reduce-scatter
            G = [[synth.grad_bf16_bits(i, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
            GT = [[torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in g] for g in G]
            for l in layers:
                l.sharded_grad_flat().zero_()
            if i % 2 == 0:
                S = layers[0].S
                recv = [torch.empty(W * S + 64, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
                for q, l in enumerate(layers):
                    F.stage_rs_scatter(l, GT[q], recv)
                for r, l in enumerate(layers):
                    F.stage_rs_recv_reduce(l, recv[r], torch.bfloat16)
            else:
                soffs, stot = F.grad_staging_layout(layers[0])
                stag = [torch.zeros(stot + 64, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
                for q, l in enumerate(layers):
                    F.stage_grads_to_staging(l, GT[q], stag[q])
                for l in layers:
                    F.stage_rs_pull(l, stag, torch.bfloat16)
            ref = w.reduce_scatter_grads(G, BF16, True)
            for r, l in enumerate(layers):
                for p in range(len(shapes)):
                    np.testing.assert_array_equal(l.sharded_grad(p).cpu().numpy().view(np.uint32),
                                                  ref[r]["order"][p].astype(np.float32).view(np.uint32),
                                                  err_msg=f"case {i} rs r={r} param {p}")
        finally:
            torch.cuda.synchronize()
            for l in layers:
                l.destroy()
