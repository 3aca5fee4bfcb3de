"""GPU parity of the HSDP world pull on ONE GPU (appendix:hsdp).

On one NVSwitch domain the HSDP reduce-scatter is one pull over all R x Ws ranks: each rank
reads its shard rows of every rank's staged grads, divides by R*Ws and sums them shard ranks
first, then replicas — the shard-group reduce-scatter and the replica all-reduce of P:476 in
one kernel (include/fsdp_b200.h, fsdp_mesh_init_hsdp).  Here the R*Ws "ranks" live on cuda:0:
Ws communicator-less meshes (one per shard rank; every replica of a shard rank has the same
layout) and R*Ws stagings, through fsdp_stage_rs_pull_hsdp — the kernels the multi-GPU path
runs over NVLink, minus the world handshakes (tests/mgpu_worker.py covers those).
The default two-phase form (replica q computes piece q of the shard into its fp32 result
buffer, fsdp_stage_hsdp_piece_pull; every replica then gathers the R pieces,
fsdp_stage_hsdp_replica_gather) is checked the same way, plus: phase 1 writes nothing
outside its piece.
Bar: bit-exact to the oracle's nested order (oracle.HsdpWorld 'order'), for the bulk (TMA)
and register pull variants, every (R, Ws) with R*Ws <= 8, ragged units, accumulation, and
one full Llama 3.1 8B block at R x Ws = 2 x 4."""
import os

import numpy as np
import pytest
import torch

import synth
from oracle import HsdpWorld
from oracle.world import BF16, FP32

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F

from test_gpu_parity import _unit, _params, KINDS  # noqa: E402

PAIRS = [(2, 1), (4, 1), (8, 1), (2, 2), (4, 2), (3, 2), (2, 3), (2, 4)]   # (R, Ws)


class _Emu:
    """Ws communicator-less meshes on cuda:0 (one per shard rank)."""

    def __init__(self, shapes, elig, Ws, params, variant=None):
        old = os.environ.get("FSDP_B200_VARIANT")
        if variant is not None:
            os.environ["FSDP_B200_VARIANT"] = str(variant)
        try:
            self.meshes = [F.Mesh(Ws, r, 0, local=True) for r in range(Ws)]
        finally:
            if variant is not None:
                if old is None:
                    del os.environ["FSDP_B200_VARIANT"]
                else:
                    os.environ["FSDP_B200_VARIANT"] = old
        self.layers = [F.fsdp_shard(m, params, elig) for m in self.meshes]

    def close(self):
        for m in self.meshes:
            m.destroy()


def _grads(seed, shapes, Wt, gd):
    if gd == BF16:
        G = [[synth.grad_bf16_bits(seed, p, g, s) for p, s in enumerate(shapes)] for g in range(Wt)]
        GT = [[torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in gg] for gg in G]
        return G, GT, torch.bfloat16
    G = [[synth.grad_fp32(seed, p, g, s) for p, s in enumerate(shapes)] for g in range(Wt)]
    GT = [[torch.from_numpy(x).cuda() for x in gg] for gg in G]
    return G, GT, torch.float32


def _run(shapes, elig, R, Ws, G, GT, tdt, mean, acc, seed, variant=None):
    Wt = R * Ws
    h = HsdpWorld(shapes, R, Ws, elig)
    emu = _Emu(shapes, elig, Ws, _params(shapes, seed), variant)
    try:
        offs, total = F.grad_staging_layout(emu.layers[0])
        stag = [torch.zeros(total + 64, dtype=tdt, device="cuda") for _ in range(Wt)]
        for g in range(Wt):   # global rank g = replica * Ws + shard rank (R15)
            F.stage_grads_to_staging(emu.layers[g % Ws], GT[g], stag[g])
        rng = np.random.default_rng(seed + 7)
        old = [rng.standard_normal(l.S).astype(np.float32) for l in emu.layers]
        for s, l in enumerate(emu.layers):
            l.sharded_grad_flat().copy_(torch.from_numpy(old[s]).cuda())
            F.stage_rs_pull_hsdp(l, stag, R, tdt, torch.float32, mean, acc)
        torch.cuda.synchronize()
        ref = h.reduce_scatter_grads(G, BF16 if tdt == torch.bfloat16 else FP32, mean)
        for s, l in enumerate(emu.layers):
            for rep in range(R):   # every replica of shard rank s holds the same result
                g = rep * Ws + s
                for p in range(len(shapes)):
                    want = ref[g]["order"][p]
                    got = l.sharded_grad(p).cpu().numpy()
                    if acc:
                        m = l.metas[p]
                        prev = old[s][m["elem_offset"]:m["elem_offset"] + got.size].reshape(got.shape)
                        want = (prev + want).astype(np.float32)
                    np.testing.assert_array_equal(got.view(np.uint32), want.astype(np.float32).view(np.uint32),
                                                  err_msg=f"R={R} Ws={Ws} shard {s} p{p}")
            flat = l.sharded_grad_flat().cpu().numpy()   # guard band: padding untouched
            real = np.zeros(l.S, dtype=bool)
            for m in l.metas:
                real[m["elem_offset"]:m["elem_offset"] + m["row_count"] * m["rest"]] = True
            np.testing.assert_array_equal(flat[~real].view(np.uint32), old[s][~real].view(np.uint32))
    finally:
        emu.close()


def _run2(shapes, elig, R, Ws, G, GT, tdt, mean, acc, seed, variant=None):
    """Two-phase: phase 1 for every global rank g into res[g], phase 2 for every replica of
    every shard rank (the emulated shard rank's grad buffer is reset before each)."""
    Wt = R * Ws
    h = HsdpWorld(shapes, R, Ws, elig)
    emu = _Emu(shapes, elig, Ws, _params(shapes, seed), variant)
    try:
        offs, total = F.grad_staging_layout(emu.layers[0])
        stag = [torch.zeros(total + 64, dtype=tdt, device="cuda") for _ in range(Wt)]
        for g in range(Wt):
            F.stage_grads_to_staging(emu.layers[g % Ws], GT[g], stag[g])
        S = emu.layers[0].S
        nan = np.uint32(0x7FC00001)
        res = [torch.full((S + 16,), int(nan), dtype=torch.int32, device="cuda").view(torch.float32)
               for _ in range(Wt)]
        for g in range(Wt):
            F.stage_hsdp_piece_pull(emu.layers[g % Ws], stag, R, g // Ws, tdt, res[g], mean=mean)
        torch.cuda.synchronize()
        P = -(-max(S, 1) // R)
        P = -(-P // 16) * 16
        for g in range(Wt):   # phase 1 wrote only inside piece g // Ws
            q = g // Ws
            r = res[g].view(torch.int32).cpu().numpy().view(np.uint32)
            outside = np.ones(S + 16, dtype=bool)
            outside[q * P:min((q + 1) * P, S)] = False
            assert np.all(r[outside] == nan), f"R={R} Ws={Ws} g={g}: write outside piece {q}"
        ref = h.reduce_scatter_grads(G, BF16 if tdt == torch.bfloat16 else FP32, mean)
        rng = np.random.default_rng(seed + 7)
        old = [rng.standard_normal(l.S).astype(np.float32) for l in emu.layers]
        for s, l in enumerate(emu.layers):
            for rep in range(R):
                l.sharded_grad_flat().copy_(torch.from_numpy(old[s]).cuda())
                F.stage_hsdp_replica_gather(l, [res[q * Ws + s] for q in range(R)], accumulate=acc)
                torch.cuda.synchronize()
                g = rep * Ws + s
                for p in range(len(shapes)):
                    want = ref[g]["order"][p]
                    got = l.sharded_grad(p).cpu().numpy()
                    if acc:
                        m = l.metas[p]
                        prev = old[s][m["elem_offset"]:m["elem_offset"] + got.size].reshape(got.shape)
                        want = (prev + want).astype(np.float32)
                    np.testing.assert_array_equal(got.view(np.uint32), want.astype(np.float32).view(np.uint32),
                                                  err_msg=f"two-phase R={R} Ws={Ws} shard {s} rep {rep} p{p}")
                flat = l.sharded_grad_flat().cpu().numpy()
                real = np.zeros(l.S, dtype=bool)
                for m in l.metas:
                    real[m["elem_offset"]:m["elem_offset"] + m["row_count"] * m["rest"]] = True
                np.testing.assert_array_equal(flat[~real].view(np.uint32), old[s][~real].view(np.uint32))
    finally:
        emu.close()


@pytest.mark.parametrize("kind,seed", KINDS[:4])
@pytest.mark.parametrize("R,Ws", PAIRS)
@pytest.mark.parametrize("variant", [None, 13])
def test_hsdp_two_phase_emulated(kind, seed, R, Ws, variant):
    shapes, elig = _unit(kind, seed, Ws)
    G, GT, tdt = _grads(seed + 40, shapes, R * Ws, BF16)
    _run2(shapes, elig, R, Ws, G, GT, tdt, True, False, seed, variant)


@pytest.mark.parametrize("R,Ws", [(2, 2), (4, 2), (2, 3), (8, 1)])
@pytest.mark.parametrize("gd,mean,acc", [(FP32, True, False), (BF16, False, False), (BF16, True, True)])
def test_hsdp_two_phase_dtypes_mean_accumulate(R, Ws, gd, mean, acc):
    shapes, elig = _unit("ragged", 8, Ws)
    G, GT, tdt = _grads(8, shapes, R * Ws, gd)
    _run2(shapes, elig, R, Ws, G, GT, tdt, mean, acc, 8)


@pytest.mark.parametrize("kind,seed", KINDS[:4])
@pytest.mark.parametrize("R,Ws", PAIRS)
@pytest.mark.parametrize("variant", [None, 13])   # default (TMA bulk pull) / register pull (VEC 8)
def test_hsdp_world_pull_emulated(kind, seed, R, Ws, variant):
    shapes, elig = _unit(kind, seed, Ws)
    G, GT, tdt = _grads(seed, shapes, R * Ws, BF16)
    _run(shapes, elig, R, Ws, G, GT, tdt, True, False, seed, variant)


@pytest.mark.parametrize("R,Ws", [(2, 2), (4, 2), (2, 3)])
@pytest.mark.parametrize("gd,mean,acc", [(FP32, True, False), (BF16, False, False), (BF16, True, True)])
def test_hsdp_world_pull_dtypes_mean_accumulate(R, Ws, gd, mean, acc):
    shapes, elig = _unit("ragged", 6, Ws)
    G, GT, tdt = _grads(6, shapes, R * Ws, gd)
    _run(shapes, elig, R, Ws, G, GT, tdt, mean, acc, 6)


def test_hsdp_world_pull_nested_differs_from_flat():
    """The nested order is a different rounding from the flat ascending sum: on data built to
    tell them apart the kernel matches the nested oracle and not the flat one (so a flat pull
    over R*Ws ranks would fail the tests above)."""
    R, Ws = 2, 2
    shapes, elig = [(64, 8)], [False]
    # terms 1, 2^-25, -1, 2^-25 (ranks 0..3; bf16-exact, mean off): flat ((1 + e) - 1) + e = e,
    # nested (1 + e) + (-1 + e) = 1 + (-1) = 0 (-1 + 2^-25 is a tie, rounded to even: -1)
    vals = [1.0, 2.0 ** -25, -1.0, 2.0 ** -25]
    G = [[(np.full(shapes[0], np.float32(v)).view(np.uint32) >> 16).astype(np.uint16)] for v in vals]
    GT = [[torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in gg] for gg in G]
    h = HsdpWorld(shapes, R, Ws, elig)
    ref = h.reduce_scatter_grads(G, BF16, False)
    x = [np.float32(v) for v in vals]
    flat = np.float32(np.float32(np.float32(x[0] + x[1]) + x[2]) + x[3])
    nested = np.float32(np.float32(x[0] + x[1]) + np.float32(x[2] + x[3]))
    assert flat != nested and np.all(ref[0]["order"][0] == nested)
    _run(shapes, elig, R, Ws, G, GT, torch.bfloat16, False, False, 0)


def test_hsdp_world_pull_full_block():
    """One full Llama 3.1 8B TransformerBlock (218.1M params) at R x Ws = 2 x 4 (Wt = 8, the
    8-GPU HSDP shape of one box): every shard rank's fp32 grad equals the nested-order oracle
    bit for bit, all elements."""
    try:
        import psutil
        if psutil.virtual_memory().available / 2 ** 30 < 40:
            pytest.skip("needs ~40 GB of free host RAM for the oracle")
    except ImportError:
        pass
    R, Ws = 2, 4
    u = synth.model_units("llama3.1-8b", include_root=False)[0]
    shapes, elig = [s for _, s, _ in u], [e for _, _, e in u]
    P_dev = [torch.zeros(s, device="cuda") for s in shapes]
    emu = _Emu(shapes, elig, Ws, P_dev)
    del P_dev
    h = HsdpWorld(shapes, R, Ws, elig)
    try:
        gen = torch.Generator(device="cuda")
        GT = []
        for g in range(R * Ws):
            gen.manual_seed(900 + g)
            GT.append([(torch.randn(s, generator=gen, device="cuda") * 1e-3).to(torch.bfloat16) for s in shapes])
        G = [[x.view(torch.int16).cpu().numpy().view(np.uint16) for x in gg] for gg in GT]
        order = [r["order"] for r in h.reduce_scatter_grads(G, BF16, True)]
        del G
        offs, total = F.grad_staging_layout(emu.layers[0])
        stag = [torch.empty(total + 64, dtype=torch.bfloat16, device="cuda") for _ in range(R * Ws)]
        for g in range(R * Ws):
            F.stage_grads_to_staging(emu.layers[g % Ws], GT[g], stag[g])
        del GT
        for s, l in enumerate(emu.layers):
            l.sharded_grad_flat().fill_(float("nan"))
            F.stage_rs_pull_hsdp(l, stag, R, torch.bfloat16, torch.float32, True, False)
        torch.cuda.synchronize()
        for s, l in enumerate(emu.layers):
            for p in range(len(shapes)):
                want = torch.from_numpy(order[s][p].view(np.int32)).cuda()
                got = l.sharded_grad(p).view(torch.int32)
                bad = (got != want).nonzero()
                assert bad.numel() == 0, f"shard {s} p{p}: {bad.shape[0]} elements differ"
        # two-phase (the default): every replica's piece, then each shard rank gathers them
        S = emu.layers[0].S
        res = [torch.empty(S + 16, dtype=torch.float32, device="cuda") for _ in range(R * Ws)]
        for g in range(R * Ws):
            F.stage_hsdp_piece_pull(emu.layers[g % Ws], stag, R, g // Ws, torch.bfloat16, res[g])
        for s, l in enumerate(emu.layers):
            l.sharded_grad_flat().fill_(float("nan"))
            F.stage_hsdp_replica_gather(l, [res[q * Ws + s] for q in range(R)])
        torch.cuda.synchronize()
        for s, l in enumerate(emu.layers):
            for p in range(len(shapes)):
                want = torch.from_numpy(order[s][p].view(np.int32)).cuda()
                got = l.sharded_grad(p).view(torch.int32)
                bad = (got != want).nonzero()
                assert bad.numel() == 0, f"two-phase shard {s} p{p}: {bad.shape[0]} elements differ"
    finally:
        emu.close()
