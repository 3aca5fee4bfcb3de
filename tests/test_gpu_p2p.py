"""GPU parity of the fused peer-memory kernels (FSDP_ALGO_P2P) on ONE GPU.

The push (unshard) and pull (reduce-scatter) kernels take arrays of W buffers; here all W
"ranks" live on cuda:0 (communicator-less meshes), every rank's push fills all W arenas,
every rank's pull reads all W stagings — the same kernels the multi-GPU path runs over
NVLink, minus the flag handshakes (which need W GPUs, tests/test_multigpu.py).
Bar: bit-exact vs the oracle for the unshard (bf16 / e4m3 given the scale) and for the
ascending-rank fp32 reduce-scatter sum."""
import numpy as np
import pytest
import torch

import synth
from oracle import World, bf16_rne_bits, bf16_bits_to_f32
from oracle.world import BF16, FP8, FP32

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F

from test_gpu_parity import _unit, _params, Emu, KINDS  # noqa: E402


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("fp8", [False, True])
def test_unshard_push_emulated(kind, seed, W, fp8):
    shapes, elig = _unit(kind, seed, W)
    P = _params(shapes, seed, edge=(seed % 2 == 1))
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, P)
    try:
        shards = w.shard(P)
        dt = torch.float8_e4m3fn if fp8 else torch.bfloat16
        scale = w.precompute_fp8_scales(shards)[1] if fp8 else None
        offs, total = F.unsharded_layout(emu.layers[0], dt)
        arenas = [torch.full((total + 16,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(W)]
        sdev = torch.from_numpy(scale).cuda() if fp8 else None
        fused = torch.zeros(max(len(shapes), 1), dtype=torch.float32, device="cuda")
        for r in range(W):
            F.stage_unshard_push(emu.layers[r], dt, arenas, fp8_scales=sdev, amax_accum=fused if fp8 else None)
        torch.cuda.synchronize()
        if fp8:   # the delayed-scaling amax fused into the push == the oracle's amax (eligible params)
            amax = w.precompute_fp8_scales(shards)[0]
            want_f = np.where(np.array(elig, bool), amax, np.float32(0)).astype(np.float32)
            np.testing.assert_array_equal(fused.cpu().numpy()[:len(shapes)].view(np.uint32), want_f.view(np.uint32))
        _, fulls = w.unshard(shards, FP8 if fp8 else BF16, scale)
        for d in range(W):
            a = arenas[d].cpu().numpy()
            written = np.zeros(a.size, dtype=bool)
            for p, want in enumerate(fulls):
                nb = want.size * want.itemsize
                got = a[offs[p]:offs[p] + nb].view(want.dtype).reshape(want.shape)
                np.testing.assert_array_equal(got, want)
                written[offs[p]:offs[p] + nb] = True
            # guard band: no byte outside the params' tensors (alignment gaps, tail) was written
            assert np.all(a[~written] == 0xA5)
    finally:
        emu.close()


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("gd,rd,mean,acc", [(BF16, FP32, True, False), (FP32, FP32, True, False),
                                            (BF16, FP32, False, False), (BF16, FP32, True, True),
                                            (BF16, BF16, True, False)])
def test_rs_pull_emulated(kind, seed, W, gd, rd, mean, acc):
    shapes, elig = _unit(kind, seed, W)
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, _params(shapes, seed))
    try:
        if gd == BF16:
            G = [[synth.grad_bf16_bits(seed, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
            GT = [[torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in g] for g in G]
            tdt = torch.bfloat16
        else:
            G = [[synth.grad_fp32(seed, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
            GT = [[torch.from_numpy(x).cuda() for x in g] for g in G]
            tdt = torch.float32
        offs, total = F.grad_staging_layout(emu.layers[0])
        stag = [torch.zeros(total + 64, dtype=tdt, device="cuda") for _ in range(W)]
        for q in range(W):
            F.stage_grads_to_staging(emu.layers[q], GT[q], stag[q])
        torch.cuda.synchronize()
        for q in (0, W - 1):   # staging holds the full grads at the published offsets
            for p, g in enumerate(GT[q]):
                np.testing.assert_array_equal(stag[q][offs[p]:offs[p] + g.numel()].view(torch.uint8).cpu().numpy(),
                                              g.reshape(-1).view(torch.uint8).cpu().numpy())
        rng = np.random.default_rng(seed)
        old = [rng.standard_normal(l.S).astype(np.float32) for l in emu.layers]
        for r, l in enumerate(emu.layers):
            l.sharded_grad_flat().copy_(torch.from_numpy(old[r]).cuda())
            F.stage_rs_pull(l, stag, tdt, torch.float32 if rd == FP32 else torch.bfloat16, mean, acc)
        torch.cuda.synchronize()
        ref = w.reduce_scatter_grads(G, gd, mean, reduce_dtype=rd)
        for r, l in enumerate(emu.layers):
            for p in range(len(shapes)):
                want = ref[r]["order"][p]
                if rd == BF16:   # the pull rounds the fp32 sum of bf16 terms to bf16
                    want = bf16_bits_to_f32(bf16_rne_bits(want.reshape(-1))).reshape(want.shape)
                got = l.sharded_grad(p).cpu().numpy()
                if acc:
                    m = l.metas[p]
                    prev = old[r][m["elem_offset"]:m["elem_offset"] + got.size].reshape(got.shape)
                    want = (prev + want).astype(np.float32)
                np.testing.assert_array_equal(got.view(np.uint32), want.astype(np.float32).view(np.uint32))
            # guard band: padding rows and alignment gaps of the grad buffer are untouched
            flat = l.sharded_grad_flat().cpu().numpy()
            real = np.zeros(l.S, dtype=bool)
            for m in l.metas:
                real[m["elem_offset"]:m["elem_offset"] + m["row_count"] * m["rest"]] = True
            np.testing.assert_array_equal(flat[~real].view(np.uint32), old[r][~real].view(np.uint32))
    finally:
        emu.close()


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("gd,rd,mean,acc", [(BF16, FP32, True, False), (FP32, FP32, True, False),
                                            (BF16, FP32, False, False), (BF16, FP32, True, True),
                                            (BF16, BF16, True, False)])
@pytest.mark.parametrize("own", [False, True])
def test_rs_store_emulated(kind, seed, W, gd, rd, mean, acc, own):
    """Store-based reduce-scatter (FSDP_P2P_RS_STORE): every rank's scatter kernel writes its
    rows of rank r's chunk into r's receive buffer at slot q (bytes checked, guard bands
    untouched), then every rank's local reduce gives the same bits as the pull.  own=True is
    the default P2P path: the scatter skips the own chunk (own slot left untouched) and the
    reduce reads the own rows from the rank's grads — same bits."""
    shapes, elig = _unit(kind, seed, W)
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, _params(shapes, seed))
    try:
        if gd == BF16:
            G = [[synth.grad_bf16_bits(seed, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
            GT = [[torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in g] for g in G]
            tdt, es = torch.bfloat16, 2
        else:
            G = [[synth.grad_fp32(seed, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
            GT = [[torch.from_numpy(x).cuda() for x in g] for g in G]
            tdt, es = torch.float32, 4
        S = emu.layers[0].S
        nbytes = W * S * es
        recv = [torch.full((nbytes + 64,), 0x5A, dtype=torch.uint8, device="cuda") for _ in range(W)]
        for q in range(W):
            F.stage_rs_scatter(emu.layers[q], GT[q], recv, include_self=not own)
        torch.cuda.synchronize()
        for r in range(W):   # slot q of rank r's buffer holds rank q's rows of r's chunk, nothing else
            a = recv[r].cpu().numpy()
            written = np.zeros(a.size, dtype=bool)
            for q in range(W):
                if own and q == r:
                    continue      # own slot never written
                for p, m in enumerate(emu.layers[r].metas):
                    cnt = m["row_count"] * m["rest"]
                    lo = (q * S + m["elem_offset"]) * es
                    want = GT[q][p].reshape(-1)[m["row_begin"] * m["rest"]:m["row_begin"] * m["rest"] + cnt]
                    np.testing.assert_array_equal(a[lo:lo + cnt * es], want.view(torch.uint8).cpu().numpy())
                    written[lo:lo + cnt * es] = True
            assert np.all(a[~written] == 0x5A)
        rng = np.random.default_rng(seed)
        old = [rng.standard_normal(l.S).astype(np.float32) for l in emu.layers]
        aligned = all(m["row_count"] == 0 or (m["row_begin"] * m["rest"] * es) % 16 == 0
                      for l in emu.layers for m in l.metas)
        for r, l in enumerate(emu.layers):
            l.sharded_grad_flat().copy_(torch.from_numpy(old[r]).cuda())
            rdt = torch.float32 if rd == FP32 else torch.bfloat16
            if own and not all(m["row_count"] == 0 or (m["row_begin"] * m["rest"] * es) % 16 == 0 for m in l.metas):
                with pytest.raises(F.FsdpError) as e:   # own-row offsets misaligned: refused, not wrong
                    F.stage_rs_recv_reduce(l, recv[r], tdt, rdt, mean, acc, own_grads=GT[r])
                assert e.value.status_name == "FSDP_ERR_INVALID_ARGUMENT"
                continue
            F.stage_rs_recv_reduce(l, recv[r], tdt, rdt, mean, acc, own_grads=GT[r] if own else None)
        torch.cuda.synchronize()
        if own and not aligned:
            return
        ref = w.reduce_scatter_grads(G, gd, mean, reduce_dtype=rd)
        for r, l in enumerate(emu.layers):
            for p in range(len(shapes)):
                want = ref[r]["order"][p]
                if rd == BF16:
                    want = bf16_bits_to_f32(bf16_rne_bits(want.reshape(-1))).reshape(want.shape)
                got = l.sharded_grad(p).cpu().numpy()
                if acc:
                    m = l.metas[p]
                    prev = old[r][m["elem_offset"]:m["elem_offset"] + got.size].reshape(got.shape)
                    want = (prev + want).astype(np.float32)
                np.testing.assert_array_equal(got.view(np.uint32), want.astype(np.float32).view(np.uint32))
            flat = l.sharded_grad_flat().cpu().numpy()
            real = np.zeros(l.S, dtype=bool)
            for m in l.metas:
                real[m["elem_offset"]:m["elem_offset"] + m["row_count"] * m["rest"]] = True
            np.testing.assert_array_equal(flat[~real].view(np.uint32), old[r][~real].view(np.uint32))
    finally:
        emu.close()
