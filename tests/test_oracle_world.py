"""Pins for oracle/world.py — CPU only.

* unshard closed form: full_p == cast(P_p), independent of W (SPEC.md:195
  "all_gather o shard == identity"), checked against torch CPU casts of the FULL tensor
  (never through the shards);
* SPEC worked examples for all-gather / reduce-scatter / all-reduce;
* amax == max |P| over the full tensor;
* reduce-scatter == brute-force sum/world of the per-rank full grads chunked by dim 0
  (BASELINE.json), bit-exact on dyadic data for any order, and within the R10 bound
  on normal data (exact reference via math.fsum on a sample)."""
import json
import math
import os

import numpy as np
import pytest
import torch

import synth
from oracle import World, bf16_bits_to_f32, e4m3_decode
from oracle.world import rs_error_ok, BF16, FP8, FP32
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SPEC = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))


def _unit(kind, seed=0, W=8):
    if kind == "toy":
        u = synth.model_units("toy", include_root=False)[0]
    else:
        u = synth.ragged_unit(seed, world_size=W)
    return [s for _, s, _ in u], [e for _, _, e in u]


def _params(shapes, unit=0):
    return [synth.param_values(unit, p, s) for p, s in enumerate(shapes)]


def test_spec_all_gather_example():
    ex = SPEC["all_gather_rank_ids"]
    W = ex["world_size"]
    w = World([(W,)], W)
    shards = w.shard([np.arange(W, dtype=np.float32)])
    _, fulls = w.unshard(shards, BF16)
    np.testing.assert_array_equal(bf16_bits_to_f32(fulls[0]), np.array(ex["result"], np.float32))


def test_spec_reduce_scatter_example():
    ex = SPEC["reduce_scatter_two_ranks"]
    w = World([(2,)], 2)
    grads = [[np.array(v, np.float32)] for v in ex["inputs"]]
    res = w.reduce_scatter_grads(grads, grad_dtype=FP32, mean=False)
    for r, want in enumerate(ex["outputs"]):
        np.testing.assert_array_equal(res[r]["order"][0], np.array(want, np.float32))
        np.testing.assert_array_equal(res[r]["exact"][0], np.array(want, np.float32))


def test_spec_rs_then_ag_is_all_reduce():
    """SPEC.md:195 algebra with SPEC.md:162's example: each of 4 ranks holds [r] (as a
    4-row grad) -> RS(sum) then AG gives 6 everywhere."""
    ex = SPEC["all_reduce_sum_rank_ids"]
    W = ex["world_size"]
    w = World([(W,)], W)
    grads = [[np.full(W, r, np.float32)] for r in range(W)]
    res = w.reduce_scatter_grads(grads, grad_dtype=FP32, mean=False)
    gathered = np.concatenate([res[r]["order"][0] for r in range(W)])
    np.testing.assert_array_equal(gathered, np.full(W, ex["result"], np.float32))


@pytest.mark.parametrize("kind,seed", [("toy", 0), ("ragged", 1), ("ragged", 2), ("ragged", 3)])
def test_unshard_bf16_closed_form_and_w_invariance(kind, seed):
    shapes, elig = _unit(kind, seed)
    P = _params(shapes, seed)
    want = [torch.from_numpy(p).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16) for p in P]
    for W in (1, 2, 3, 4, 5, 8):
        w = World(shapes, W, elig)
        ag, fulls = w.unshard(w.shard(P), BF16)
        assert ag.size == W * 2 * w.S
        for f, g in zip(fulls, want):
            assert f.shape == g.shape
            np.testing.assert_array_equal(f, g)


@pytest.mark.parametrize("kind,seed", [("toy", 0), ("ragged", 4), ("ragged", 5)])
def test_unshard_fp8_closed_form(kind, seed):
    shapes, elig = _unit(kind, seed)
    P = _params(shapes, seed)
    for W in (1, 2, 3, 8):
        w = World(shapes, W, elig)
        shards = w.shard(P)
        amax, scale = w.precompute_fp8_scales(shards)
        for p, (full, e) in enumerate(zip(P, elig)):
            if e:
                assert amax[p] == (np.abs(full).max() if full.size else 0.0)  # over the FULL tensor
                assert scale[p] == np.float32(448.0 / np.float64(max(amax[p], np.float32(1e-12))))
        ag, fulls = w.unshard(shards, FP8, scale)
        assert ag.size == W * w.S_bytes_fp8
        for p, (f, full, e) in enumerate(zip(fulls, P, elig)):
            t = torch.from_numpy(full)
            if e:
                ref = (t * torch.tensor(scale[p])).clamp(-448, 448).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
                assert f.dtype == np.uint8
            else:
                ref = t.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
            np.testing.assert_array_equal(f, ref)


def _brute_rs(grads_per_rank, shapes, W, mean, widen):
    """Sum of the full grads over ranks in fp64 (exact for dyadic data), divided by W,
    then chunked on dim 0 with torch.chunk (library split)."""
    outs = [[None] * len(shapes) for _ in range(W)]
    for p, shape in enumerate(shapes):
        tot = np.zeros(shape, np.float64)
        for q in range(W):
            tot += widen(grads_per_rank[q][p]).astype(np.float64)
        if mean:
            tot = tot / W
        if shape[0] == 0:
            chunks = []
        else:
            chunks = list(torch.chunk(torch.from_numpy(tot), W, dim=0))
        for r in range(W):
            c = chunks[r].numpy() if r < len(chunks) else np.zeros((0,) + shape[1:])
            outs[r][p] = c
    return outs


@pytest.mark.parametrize("W", [1, 2, 4, 8])
@pytest.mark.parametrize("kind,seed", [("toy", 0), ("ragged", 6), ("ragged", 7)])
def test_rs_dyadic_bitexact_any_order(W, kind, seed):
    shapes, elig = _unit(kind, seed, W)
    w = World(shapes, W, elig)
    grads = [[synth.dyadic_grad_bf16_bits(seed, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
    res = w.reduce_scatter_grads(grads, BF16, mean=True)
    brute = _brute_rs(grads, shapes, W, True, bf16_bits_to_f32)
    for r in range(W):
        for p in range(len(shapes)):
            want = brute[r][p].astype(np.float32)
            np.testing.assert_array_equal(res[r]["order"][p], want)
            np.testing.assert_array_equal(res[r]["exact"][p], want)
            # reversed order gives the same bits (order independence on dyadic data)
            assert res[r]["order"][p].shape == want.shape


@pytest.mark.parametrize("W", [2, 3, 8])
def test_rs_normal_data_exact_reference_and_bound(W):
    shapes, elig = _unit("ragged", 8, W)
    w = World(shapes, W, elig)
    grads = [[synth.grad_bf16_bits(8, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
    res = w.reduce_scatter_grads(grads, BF16, mean=True)
    rng = np.random.default_rng(0)
    for r in range(W):
        for p, shape in enumerate(shapes):
            ex = res[r]["exact"][p].reshape(-1)
            od = res[r]["order"][p].reshape(-1)
            mg = res[r]["mag"][p].reshape(-1)
            ok, ratio, _ = rs_error_ok(od, ex, mg, W)
            assert ratio <= 1.0
            if ex.size:
                # exact reference by math.fsum on sampled elements (brute force)
                m = w.layouts[r].params[p]
                for k in rng.integers(0, ex.size, size=min(50, ex.size)):
                    vals = [float(bf16_bits_to_f32(grads[q][p].reshape(-1)[r * m.padded_numel + k:r * m.padded_numel + k + 1])[0]
                                  / np.float32(W)) for q in range(W)]
                    vals32 = [float(np.float32(v)) for v in vals]
                    assert ex[k] == np.float32(math.fsum(vals32))
    if W == 2:   # two-term fp32 sums are commutative and correctly rounded
        for r in range(W):
            for p in range(len(shapes)):
                np.testing.assert_array_equal(res[r]["order"][p], res[r]["exact"][p])


def test_rs_mean_false_and_w1_identity():
    shapes, elig = _unit("toy")
    w = World(shapes, 1, elig)
    g = [synth.grad_bf16_bits(0, p, 0, s) for p, s in enumerate(shapes)]
    res = w.reduce_scatter_grads([g], BF16, mean=True)
    for p in range(len(shapes)):
        np.testing.assert_array_equal(res[0]["order"][p], bf16_bits_to_f32(g[p]).reshape(shapes[p]))


def test_rs_copy_out_shapes_empty_shards():
    shapes = [(3, 5), (1,), (10, 2)]
    w = World(shapes, 4)
    out = np.arange(w.S, dtype=np.float32)
    for r in range(4):
        got = w.rs_copy_out(out, r)
        for m, g in zip(w.layouts[r].params, got):
            assert g.shape == (m.row_count,) + m.shape[1:]
    assert w.rs_copy_out(out, 3)[0].shape == (0, 5)      # d0=3 over 4 ranks -> rank 3 empty
    assert w.rs_copy_out(out, 1)[1].shape == (0,)


def test_rs_bf16_reduce_bound():
    W = 4
    shapes, elig = _unit("ragged", 9, W)
    w = World(shapes, W, elig)
    grads = [[synth.grad_bf16_bits(9, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
    res = w.reduce_scatter_grads(grads, BF16, mean=True, reduce_dtype=BF16)
    ref = w.reduce_scatter_grads(grads, BF16, mean=True, reduce_dtype=FP32)
    for r in range(W):
        for p in range(len(shapes)):
            ok, ratio, nrel = rs_error_ok(res[r]["order"][p].reshape(-1), ref[r]["exact"][p].reshape(-1),
                                          ref[r]["mag"][p].reshape(-1), W, rel=(W - 1) * 2.0 ** -8 + 2.0 ** -8)
            assert ratio <= 1.0


# ----------------------------------------------------------------------------- HSDP (f1)
from oracle import HsdpWorld  # noqa: E402


def _grads(kind, shapes, W, seed):
    gen = synth.dyadic_grad_bf16_bits if kind == "dyadic" else synth.grad_bf16_bits
    return [[gen(seed, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]


@pytest.mark.parametrize("R,Ws", [(1, 4), (2, 2), (2, 4), (4, 2), (4, 1)])   # W = 2^k: /W exact
def test_hsdp_rs_bruteforce_dyadic(R, Ws):
    """Sharded grad of global rank (r, s) == sum over ALL R*Ws ranks' grads / (R*Ws),
    chunked on dim 0 over the shard group (torch.chunk) — PAPER.md:476."""
    shapes, elig = _unit("ragged", 11, Ws)
    h = HsdpWorld(shapes, R, Ws, elig)
    G = _grads("dyadic", shapes, R * Ws, 11)
    res = h.reduce_scatter_grads(G, BF16, True)
    for p, shape in enumerate(shapes):
        tot = np.zeros(shape, np.float64)
        for q in range(R * Ws):
            tot += bf16_bits_to_f32(G[q][p]).astype(np.float64)
        tot /= R * Ws
        chunks = list(torch.chunk(torch.from_numpy(tot), Ws, dim=0)) if shape[0] else []
        for g in range(R * Ws):
            s = g % Ws
            want = chunks[s].numpy() if s < len(chunks) else np.zeros((0,) + shape[1:])
            np.testing.assert_array_equal(res[g]["order"][p], want.astype(np.float32))
            np.testing.assert_array_equal(res[g]["exact"][p], want.astype(np.float32))


def test_hsdp_degenerate_and_spec_cross_config():
    """R=1 is plain FSDP; "HSDP (replicate 2 x shard 2) equals FSDP 4": the
    gathered gradient of HSDP(2x2) equals FSDP(4)'s (dyadic data: exact for any order)."""
    shapes, elig = _unit("toy")
    G4 = _grads("normal", shapes, 4, 0)
    a = HsdpWorld(shapes, 1, 4, elig).reduce_scatter_grads(G4, BF16, True)
    b = World(shapes, 4, elig).reduce_scatter_grads(G4, BF16, True)
    for r in range(4):
        for p in range(len(shapes)):
            np.testing.assert_array_equal(a[r]["order"][p], b[r]["order"][p])
    G = _grads("dyadic", shapes, 4, 1)
    h = HsdpWorld(shapes, 2, 2, elig).reduce_scatter_grads(G, BF16, True)
    f = World(shapes, 4, elig).reduce_scatter_grads(G, BF16, True)
    for p in range(len(shapes)):
        full_h = np.concatenate([h[s]["order"][p] for s in range(2)])
        full_f = np.concatenate([f[r]["order"][p] for r in range(4)])
        np.testing.assert_array_equal(full_h, full_f)
        for s in range(2):   # replicas hold identical shards
            np.testing.assert_array_equal(h[s]["order"][p], h[2 + s]["order"][p])


def test_hsdp_normal_data_bound():
    shapes, elig = _unit("ragged", 12, 4)
    h = HsdpWorld(shapes, 2, 4, elig)
    res = h.reduce_scatter_grads(_grads("normal", shapes, 8, 12), BF16, True)
    for g in range(8):
        for p in range(len(shapes)):
            ok, ratio, _ = rs_error_ok(res[g]["order"][p].reshape(-1), res[g]["exact"][p].reshape(-1),
                                       res[g]["mag"][p].reshape(-1), 8)
            assert ratio <= 1.0


def test_hsdp_order_is_nested_hand_example():
    """The HSDP 'order' result is the shard-group sum (ascending shard rank) of each replica,
    then the replica partials summed ascending (reduce-scatter in the shard
    group, then the all-reduce across replicas; reading R15) — NOT the flat ascending sum
    over all R*Ws ranks.  Hand example, R = Ws = 2, mean off, terms 1, 2^-25, -1, 2^-25 for
    global ranks 0..3 (bf16-exact): nested (1 + 2^-25) + (-1 + 2^-25) = 1 + (-1) = 0 (each
    add is a tie or below half an ulp and rounds to the even neighbour), flat
    ((1 + 2^-25) - 1) + 2^-25 = 2^-25.  The device world pull is pinned to this oracle."""
    shapes, elig = [(4, 16)], [False]
    vals = [1.0, 2.0 ** -25, -1.0, 2.0 ** -25]
    G = [[(np.full(shapes[0], np.float32(v)).view(np.uint32) >> 16).astype(np.uint16)] for v in vals]
    res = HsdpWorld(shapes, 2, 2, elig).reduce_scatter_grads(G, BF16, False)
    for g in range(4):
        assert res[g]["order"][0].shape == (2, 16)
        np.testing.assert_array_equal(res[g]["order"][0].view(np.uint32), np.zeros((2, 16), np.uint32))
        # the exact sum is 2^-24 (= 2 * 2^-25), representable: 'exact' differs from 'order'
        np.testing.assert_array_equal(res[g]["exact"][0], np.full((2, 16), np.float32(2.0 ** -24)))
