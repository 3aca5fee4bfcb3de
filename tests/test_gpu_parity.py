"""GPU parity: every kernel of the hot path vs the CPU oracle, through the C ABI.

W ranks are emulated on one GPU with communicator-less meshes (fsdp_mesh_init_local):
each rank's layer runs its copy-in / amax / RS copy-in kernels, the all-gather buffer
handed to the copy-out kernel is the ORACLE's (never the CUDA path's), and the outputs are
compared element by element with the oracle.  Bar (BASELINE.json): bit-exact for the
unshard copy-in/copy-out, metadata, amax and the fp8 cast given the same scale; the RS
copy-in (fp32(g) / W) is bit-exact too (one IEEE op).  The full-path tests run the real
NCCL communicator at W = 1 (multi-GPU W > 1 lives in test_multigpu.py)."""
import numpy as np
import pytest
import torch

import synth
from oracle import World, bf16_rne_bits, e4m3_encode
from oracle.world import BF16, FP8, FP32, rs_error_ok

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F


def _unit(kind, seed=0, W=8):
    if kind == "toy":
        u = synth.model_units("toy", include_root=False)[0]
    elif kind == "toyroot":
        u = synth.model_units("toy")[-1]
    else:
        u = synth.ragged_unit(seed, world_size=W)
    return [s for _, s, _ in u], [e for _, _, e in u]


def _params(shapes, seed, edge=False):
    ps = [synth.param_values(seed, p, s) for p, s in enumerate(shapes)]
    if edge:  # splice cast-boundary values into the params
        for p, a in enumerate(ps):
            flat = a.reshape(-1)
            e = synth.edge_values(flat.size, seed * 131 + p)
            e = np.where(np.abs(e) < 3e38, e, np.float32(1.0)).astype(np.float32)
            flat[::2] = e[::2]
    return ps


def _u8(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).view(np.uint8).reshape(-1)


class Emu:
    """W communicator-less meshes on cuda:0, one layer per rank."""

    def __init__(self, shapes, elig, W, params):
        self.W = W
        self.meshes = [F.Mesh(W, r, 0, local=True) for r in range(W)]
        self.layers = [F.fsdp_shard(m, params, elig) for m in self.meshes]

    def close(self):
        for m in self.meshes:
            m.destroy()


KINDS = [("toy", 0), ("toyroot", 0), ("ragged", 1), ("ragged", 2), ("ragged", 3), ("ragged", 4), ("ragged", 5)]
WS = [1, 2, 3, 4, 5, 8]


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", WS)
def test_shard_metadata_and_contents(kind, seed, W):
    shapes, elig = _unit(kind, seed, W)
    P = _params(shapes, seed)
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, P)
    try:
        shards = w.shard(P)
        for r, l in enumerate(emu.layers):
            assert l.S == w.S
            got = l.sharded_flat().cpu().numpy()
            np.testing.assert_array_equal(got.view(np.uint32), shards[r].view(np.uint32))
    finally:
        emu.close()


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", WS)
def test_unshard_bf16_copy_in_copy_out(kind, seed, W):
    shapes, elig = _unit(kind, seed, W)
    P = _params(shapes, seed, edge=True)
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, P)
    try:
        shards = w.shard(P)
        slots = [w.copy_in(s, BF16) for s in shards]
        for r, l in enumerate(emu.layers):          # K2 copy-in, bit-exact per rank
            slot = torch.empty(2 * l.S, dtype=torch.uint8, device="cuda")
            F.stage_copy_in(l, torch.bfloat16, slot)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(slot.cpu().numpy(), slots[r])
        ag = w.all_gather(slots)                    # oracle's all-gather buffer
        fulls = w.copy_out(ag, BF16)
        ag_dev = torch.from_numpy(ag).cuda()
        for r in (0, W - 1):                         # K4 copy-out on two ranks
            outs = [torch.full(s, float("nan"), dtype=torch.bfloat16, device="cuda") for s in shapes]
            F.stage_copy_out(emu.layers[r], torch.bfloat16, ag_dev, outs)
            torch.cuda.synchronize()
            for o, want in zip(outs, fulls):
                np.testing.assert_array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), want)
    finally:
        emu.close()


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_fp8_amax_scale_copy_in_copy_out(kind, seed, W):
    shapes, elig = _unit(kind, seed, W)
    P = _params(shapes, seed, edge=(seed % 2 == 1))
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, P)
    try:
        shards = w.shard(P)
        amax, scale = w.precompute_fp8_scales(shards)
        # K1 local amax per rank (bit-exact; max is order independent)
        for r, l in enumerate(emu.layers):
            a = torch.empty(l.P, dtype=torch.float32, device="cuda")
            F.stage_local_amax(l, a)
            np.testing.assert_array_equal(a.cpu().numpy().view(np.uint32), w.local_amax(shards[r]).view(np.uint32))
        # K1b scale from the oracle's global amax
        l0 = emu.layers[0]
        s_dev = torch.empty(l0.P, dtype=torch.float32, device="cuda")
        F.stage_fp8_scale(l0, torch.from_numpy(amax.copy()).cuda(), s_dev)
        np.testing.assert_array_equal(s_dev.cpu().numpy().view(np.uint32), scale.view(np.uint32))
        # K3 copy-in given the oracle's scale, then K4 copy-out of the oracle's buffer
        scale_dev = torch.from_numpy(scale).cuda()
        slots = [w.copy_in(s, FP8, scale) for s in shards]
        fused = torch.zeros(l0.P, dtype=torch.float32, device="cuda")   # amax fused into K3 (delayed)
        for r, l in enumerate(emu.layers):
            slot = torch.zeros(l.S_bytes_fp8, dtype=torch.uint8, device="cuda")
            F.stage_copy_in(l, torch.float8_e4m3fn, slot, fp8_scales=scale_dev, amax_accum=fused)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(slot.cpu().numpy(), slots[r])
        # max over the ranks' fused accumulators == the oracle's all-reduced amax (eligible params)
        want_f = np.where(np.array(elig, bool), amax, np.float32(0)).astype(np.float32)
        np.testing.assert_array_equal(fused.cpu().numpy().view(np.uint32), want_f.view(np.uint32))
        ag = w.all_gather(slots)
        fulls = w.copy_out(ag, FP8)
        outs = [torch.empty(s, dtype=torch.float8_e4m3fn if e else torch.bfloat16, device="cuda")
                for s, e in zip(shapes, elig)]
        F.stage_copy_out(emu.layers[W - 1], torch.float8_e4m3fn, torch.from_numpy(ag).cuda(), outs)
        torch.cuda.synchronize()
        for o, want in zip(outs, fulls):
            got = o.view(torch.uint8).cpu().numpy() if o.dtype == torch.float8_e4m3fn else \
                o.view(torch.int16).cpu().numpy().view(np.uint16)
            np.testing.assert_array_equal(got, want)
    finally:
        emu.close()


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", WS)
@pytest.mark.parametrize("gd,rd,mean", [(BF16, FP32, True), (FP32, FP32, True), (BF16, FP32, False),
                                        (BF16, BF16, True)])
def test_rs_copy_in(kind, seed, W, gd, rd, mean):
    shapes, elig = _unit(kind, seed, W)
    P = _params(shapes, seed)
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, P)
    try:
        for q in (0, W - 1):
            if gd == BF16:
                g = [synth.grad_bf16_bits(seed, p, q, s) for p, s in enumerate(shapes)]
                gt = [torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in g]
            else:
                g = [synth.grad_fp32(seed, p, q, s) for p, s in enumerate(shapes)]
                gt = [torch.from_numpy(x).cuda() for x in g]
            want = w.rs_copy_in(g, gd, mean, rd)
            out = torch.full((W * w.S,), -1, dtype=torch.float32 if rd == FP32 else torch.int16, device="cuda")
            F.stage_rs_copy_in(emu.layers[q], gt, torch.float32 if rd == FP32 else torch.bfloat16, mean, out)
            torch.cuda.synchronize()
            got = out.cpu().numpy()
            np.testing.assert_array_equal(got.view(np.uint32 if rd == FP32 else np.uint16),
                                          want.view(np.uint32 if rd == FP32 else np.uint16))
    finally:
        emu.close()


@pytest.mark.parametrize("rd,acc", [(FP32, False), (FP32, True), (BF16, False), (BF16, True)])
def test_rs_copy_out(rd, acc):
    shapes, elig = _unit("ragged", 2, 4)
    w = World(shapes, 4, elig)
    emu = Emu(shapes, elig, 4, _params(shapes, 2))
    try:
        l = emu.layers[1]
        rng = np.random.default_rng(5)
        old = rng.standard_normal(w.S).astype(np.float32)
        new32 = rng.standard_normal(w.S).astype(np.float32)
        if rd == BF16:
            new = bf16_rne_bits(new32)
            new_t = torch.from_numpy(new.view(np.int16)).cuda()
            new_f = (new.astype(np.uint32) << 16).view(np.float32)
        else:
            new_t = torch.from_numpy(new32).cuda()
            new_f = new32
        l.sharded_grad_flat().copy_(torch.from_numpy(old).cuda())
        F.stage_rs_copy_out(l, new_t, torch.float32 if rd == FP32 else torch.bfloat16, acc)
        torch.cuda.synchronize()
        want = (old + new_f).astype(np.float32) if acc else new_f
        np.testing.assert_array_equal(l.sharded_grad_flat().cpu().numpy().view(np.uint32), want.view(np.uint32))
        # per-param views follow the oracle's copy-out (shape (rows, *rest), empty shards)
        for p, g in enumerate(w.rs_copy_out(want, 1)):
            np.testing.assert_array_equal(l.sharded_grad(p).cpu().numpy(), g)
    finally:
        emu.close()


# ----------------------------------------------------------------------------- full path, W=1
def _nccl_mesh_w1():
    return F.Mesh(1, 0, 0, unique_id=F.get_unique_id())


@pytest.mark.parametrize("local", [False, True])
@pytest.mark.parametrize("kind,seed", [("toy", 0), ("toyroot", 0), ("ragged", 3)])
def test_full_path_w1(local, kind, seed):
    shapes, elig = _unit(kind, seed, 1)
    P = _params(shapes, seed)
    w = World(shapes, 1, elig)
    mesh = F.Mesh(1, 0, 0, local=True) if local else _nccl_mesh_w1()
    try:
        layer = F.fsdp_shard(mesh, [torch.from_numpy(p) for p in P], elig)
        shards = w.shard(P)
        # bf16 unshard
        outs = F.all_gather_params(layer, torch.bfloat16)
        _, fulls = w.unshard(shards, BF16)
        for o, want in zip(outs, fulls):
            np.testing.assert_array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), want)
        F.fsdp_reshard(layer)
        # fp8 unshard with precomputed scales
        F.precompute_fp8_scales(mesh, [layer])
        amax, scale = w.precompute_fp8_scales(shards)
        s_dev, a_dev = layer.fp8_scales()
        np.testing.assert_array_equal(s_dev.cpu().numpy().view(np.uint32), scale.view(np.uint32))
        np.testing.assert_array_equal(a_dev.cpu().numpy().view(np.uint32), amax.view(np.uint32))
        outs = F.all_gather_params(layer, torch.float8_e4m3fn)
        _, fulls = w.unshard(shards, FP8, scale)
        for o, want in zip(outs, fulls):
            got = o.view(torch.uint8).cpu().numpy() if o.dtype == torch.float8_e4m3fn else \
                o.view(torch.int16).cpu().numpy().view(np.uint16)
            np.testing.assert_array_equal(got, want)
        F.fsdp_reshard(layer)
        # reduce-scatter (identity collective at W=1), fp32 direct and accumulate
        g = [synth.grad_bf16_bits(seed, p, 0, s) for p, s in enumerate(shapes)]
        gt = [torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in g]
        F.reduce_scatter_grads(layer, gt)
        F.fsdp_wait_reduce_scatter(layer)
        res = w.reduce_scatter_grads([g], BF16, True)[0]["order"]
        for p in range(len(shapes)):
            np.testing.assert_array_equal(layer.sharded_grad(p).cpu().numpy(), res[p])
        F.reduce_scatter_grads(layer, gt, accumulate=True)
        F.fsdp_wait_reduce_scatter(layer)
        for p in range(len(shapes)):
            np.testing.assert_array_equal(layer.sharded_grad(p).cpu().numpy(), (res[p] + res[p]).astype(np.float32))
        mesh.synchronize(60000)
    finally:
        mesh.destroy()


def test_state_errors_and_nonfinite():
    shapes, elig = _unit("toy")
    P = _params(shapes, 0)
    mesh = _nccl_mesh_w1()
    try:
        layer = F.fsdp_shard(mesh, [torch.from_numpy(p) for p in P], elig)
        with pytest.raises(F.FsdpError) as e:
            layer.unsharded_param(0)
        assert e.value.status_name == "FSDP_ERR_STATE"
        F.fsdp_unshard(layer)
        F.fsdp_unshard(layer)               # already unsharded, same dtype: no-op (FSDP2 unshard())
        with pytest.raises(F.FsdpError) as e:
            F.fsdp_unshard(layer, torch.float8_e4m3fn)   # another dtype while unsharded
        assert e.value.status_name == "FSDP_ERR_STATE"
        with pytest.raises(F.FsdpError):
            layer.unsharded_param(0)        # before wait_unshard
        F.fsdp_wait_unshard(layer)
        assert layer.unsharded_param(0).shape == shapes[0]
        F.fsdp_reshard(layer)
        F.fsdp_reshard(layer)               # idempotent
        g = [torch.zeros(s, dtype=torch.bfloat16, device="cuda") for s in shapes]
        F.reduce_scatter_grads(layer, g)
        with pytest.raises(F.FsdpError) as e:
            F.reduce_scatter_grads(layer, g)
        assert e.value.status_name == "FSDP_ERR_STATE"
        F.fsdp_wait_reduce_scatter(layer)
        with pytest.raises(F.FsdpError) as e:
            F.fsdp_unshard(layer, torch.float32)
        assert e.value.status_name == "FSDP_ERR_DTYPE"
        # non-finite amax is surfaced
        layer.sharded_param(0).view(-1)[3] = float("inf")
        F.precompute_fp8_scales(mesh, [layer])
        with pytest.raises(F.FsdpError) as e:
            mesh.synchronize(60000)
        assert e.value.status_name == "FSDP_ERR_NONFINITE"
        mesh.synchronize(60000)             # flag cleared
    finally:
        mesh.destroy()


def test_prefetch_and_stream_delays_do_not_change_results():
    """Unshard of layer i+1 issued before layer i is consumed, random delays injected on
    the compute stream, reduce-scatters in flight: results equal the serial run."""
    units = synth.model_units("toy")
    mesh = _nccl_mesh_w1()
    try:
        layers, worlds, params = [], [], []
        for u_i, u in enumerate(units):
            shapes = [s for _, s, _ in u]
            elig = [e for _, _, e in u]
            P = _params(shapes, u_i)
            params.append(P)
            worlds.append(World(shapes, 1, elig))
            layers.append(F.fsdp_shard(mesh, [torch.from_numpy(p) for p in P], elig))
        rng = np.random.default_rng(0)
        comp = torch.cuda.Stream()
        with torch.cuda.stream(comp):
            got = []
            F.fsdp_unshard(layers[0], stream=comp)
            grads = []
            for i, l in enumerate(layers):
                F.fsdp_wait_unshard(l, stream=comp)
                if i + 1 < len(layers):
                    F.fsdp_unshard(layers[i + 1], stream=comp)
                torch.cuda._sleep(int(rng.integers(1000, 200000)))
                got.append([t.clone() for t in l.unsharded_params()])
                torch.cuda._sleep(int(rng.integers(1000, 200000)))
                F.fsdp_reshard(l, stream=comp)
                g = [torch.ones(s, dtype=torch.bfloat16, device="cuda") * (i + 1) for s in l.shapes]
                grads.append(g)
                F.reduce_scatter_grads(l, g, stream=comp)
            for l in layers:
                F.fsdp_wait_reduce_scatter(l, stream=comp)
        comp.synchronize()
        for i, l in enumerate(layers):
            _, fulls = worlds[i].unshard(worlds[i].shard(params[i]), BF16)
            for t, want in zip(got[i], fulls):
                np.testing.assert_array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16), want)
            for p in range(l.P):
                assert torch.all(l.sharded_grad(p) == float(i + 1))
    finally:
        mesh.destroy()


# ----------------------------------------------------------------------------- exhaustive casts
def _cast_layer(mesh, n):
    return F.fsdp_shard(mesh, None, [True], shapes=[(n,)])


def test_bf16_cast_all_fp32_patterns():
    """All 2**32 fp32 bit patterns through K2 vs the oracle's RNE definition (NaN patterns
    excluded: outside the bit-exact domain, reading R5)."""
    n = 1 << 26
    mesh = F.Mesh(1, 0, 0, local=True)
    try:
        layer = _cast_layer(mesh, n)
        shard = layer.sharded_flat()
        slot = torch.empty(2 * layer.S, dtype=torch.uint8, device="cuda")
        base = torch.arange(n, dtype=torch.int64, device="cuda")
        for c in range(1 << 6):
            pat = ((base + c * n) & 0xFFFFFFFF).to(torch.int64)
            pat = torch.where(pat >= (1 << 31), pat - (1 << 32), pat).to(torch.int32)
            shard[:n].copy_(pat.view(torch.float32))
            F.stage_copy_in(layer, torch.bfloat16, slot)
            got = slot[:2 * n].view(torch.int16).cpu().numpy().view(np.uint16)
            x = pat.cpu().numpy().view(np.float32)
            ok = ~np.isnan(x)
            np.testing.assert_array_equal(got[ok], bf16_rne_bits(x[ok]))
    finally:
        mesh.destroy()


def test_e4m3_cast_exhaustive_vs_torch_and_sampled_vs_oracle():
    """All 2**32 patterns (scale 1) vs torch CUDA's clamp+cast (the library routine the oracle
    is pinned to); a 2**24 random sample plus every e4m3 midpoint neighbourhood vs the oracle."""
    n = 1 << 26
    mesh = F.Mesh(1, 0, 0, local=True)
    try:
        layer = _cast_layer(mesh, n)
        shard = layer.sharded_flat()
        slot = torch.empty(layer.S_bytes_fp8, dtype=torch.uint8, device="cuda")
        one = torch.ones(1, dtype=torch.float32, device="cuda")
        base = torch.arange(n, dtype=torch.int64, device="cuda")
        for c in range(1 << 6):
            pat = ((base + c * n) & 0xFFFFFFFF)
            pat = torch.where(pat >= (1 << 31), pat - (1 << 32), pat).to(torch.int32)
            x = pat.view(torch.float32)
            shard[:n].copy_(x)
            F.stage_copy_in(layer, torch.float8_e4m3fn, slot, fp8_scales=one)
            ref = x.clamp(-448.0, 448.0).to(torch.float8_e4m3fn).view(torch.uint8)
            ok = ~torch.isnan(x)
            assert torch.equal(slot[:n][ok], ref[ok]), c
        # oracle on a random sample + boundary neighbourhoods
        rng = np.random.default_rng(11)
        samp = rng.integers(0, 1 << 32, size=1 << 24, dtype=np.uint64).astype(np.uint32).view(np.float32)
        samp = np.concatenate([samp[~np.isnan(samp)], synth.edge_values(1 << 20, 3)])[:n]
        shard[:samp.size].copy_(torch.from_numpy(samp).cuda())
        F.stage_copy_in(layer, torch.float8_e4m3fn, slot, fp8_scales=one)
        got = slot[:samp.size].cpu().numpy()
        np.testing.assert_array_equal(got, e4m3_encode(samp))
    finally:
        mesh.destroy()


# ----------------------------------------------------------------------------- full size
@pytest.mark.parametrize("W", [1, 8])
def test_llama8b_block_full_size_sampled(W):
    """Llama 3.1 8B block layout at the bench's sizes: emulated W ranks on one GPU,
    copy-in (CUDA) of every rank -> copy-out; sampled elements of every full tensor vs the
    oracle's closed form bf16(P); sampled RS copy-in elements vs fp32(g)/W."""
    u = synth.model_units("llama3.1-8b", include_root=False)[0]
    shapes = [s for _, s, _ in u]
    elig = [e for _, _, e in u]
    gen = torch.Generator(device="cuda").manual_seed(1234)
    P = [torch.randn(s, generator=gen, device="cuda", dtype=torch.float32) * 0.02 for s in shapes]
    emu = Emu(shapes, elig, W, P)
    try:
        l0 = emu.layers[0]
        ag = torch.empty(W * 2 * l0.S, dtype=torch.uint8, device="cuda")
        for r, l in enumerate(emu.layers):
            F.stage_copy_in(l, torch.bfloat16, ag[r * 2 * l.S:(r + 1) * 2 * l.S])
        outs = [torch.empty(s, dtype=torch.bfloat16, device="cuda") for s in shapes]
        F.stage_copy_out(emu.layers[W - 1], torch.bfloat16, ag, outs)
        torch.cuda.synchronize()
        rng = np.random.default_rng(0)
        for p, (o, full) in enumerate(zip(outs, P)):
            idx = torch.from_numpy(rng.integers(0, full.numel(), 4096)).cuda()
            want = bf16_rne_bits(full.view(-1)[idx].cpu().numpy())
            got = o.view(-1)[idx].view(torch.int16).cpu().numpy().view(np.uint16)
            np.testing.assert_array_equal(got, want)
        # RS copy-in of rank 0's grads
        G = [(torch.randn(s, generator=gen, device="cuda") * 1e-3).to(torch.bfloat16) for s in shapes]
        rs_in = torch.empty(W * l0.S, dtype=torch.float32, device="cuda")
        F.stage_rs_copy_in(l0, G, torch.float32, True, rs_in)
        torch.cuda.synchronize()
        for p, (g, m) in enumerate(zip(G, l0.metas)):
            for r in range(W):
                mr = emu.layers[r].metas[p]
                cnt = mr["row_count"] * mr["rest"]
                k = torch.from_numpy(rng.integers(0, cnt, 2048)).cuda()
                src = g.view(-1)[r * mr["padded_numel"] + k].view(torch.int16).cpu().numpy().view(np.uint16)
                want = ((src.astype(np.uint32) << 16).view(np.float32) / np.float32(W)).astype(np.float32)
                got = rs_in[r * l0.S + mr["elem_offset"] + k].cpu().numpy()
                np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    finally:
        emu.close()
