"""GPU parity of the fp8 scaling strategies ("dynamic, delayed, and static"):
delayed scaling over an amax history vs oracle.scaling.DelayedScaling,
bit-exact scales step by step, and the fp8 unshard with those scales vs the oracle cast;
static scaling = caller scales passed to the unshard."""
import numpy as np
import pytest
import torch

from oracle import World
from oracle.scaling import DelayedScaling
from oracle.world import FP8

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F

from test_gpu_parity import _unit, _params  # noqa: E402


FACTORS = [1.0, 2.0, 0.25, 8.0, 1.0, 1.0, 1.0, 0.5, 3.0]


@pytest.mark.parametrize("H", [1, 4, 16])
@pytest.mark.parametrize("fuse", [False, True])
def test_fp8_delayed_scaling_sequence(H, fuse, monkeypatch):
    """fuse=False: a K1 amax pass at every precompute; fuse=True (the default): the amax is
    folded into the fp8 unshard's cast and recorded at the next precompute — the scales must
    be the oracle's DelayedScaling sequence bit for bit either way; the reported amax is the
    current step's (K1) or the previous step's (fused)."""
    monkeypatch.setenv("FSDP_B200_AMAX_FUSE", "1" if fuse else "0")
    shapes, elig = _unit("toy")
    P = _params(shapes, 0)
    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id())
    try:
        layer = F.fsdp_shard(mesh, [torch.from_numpy(p) for p in P], elig)
        w = World(shapes, 1, elig)
        d = DelayedScaling(len(shapes), H)
        base = layer.sharded_flat().clone()
        prev_amax = None
        for f in FACTORS:
            cur = (base * f).contiguous()
            layer.sharded_flat().copy_(cur)
            F.precompute_fp8_scales(mesh, [layer], history_len=H)
            s_dev, a_dev = layer.fp8_scales()
            shard = cur.cpu().numpy()
            amax, _ = w.precompute_fp8_scales([shard])
            want = d.step(amax, elig)
            rec = prev_amax if (fuse and prev_amax is not None) else amax
            np.testing.assert_array_equal(a_dev.cpu().numpy().view(np.uint32), rec.view(np.uint32))
            np.testing.assert_array_equal(s_dev.cpu().numpy().view(np.uint32), want.view(np.uint32))
            outs = F.all_gather_params(layer, torch.float8_e4m3fn)
            _, fulls = w.unshard([shard], FP8, want)
            for o, ref in zip(outs, fulls):
                got = o.view(torch.uint8).cpu().numpy() if o.dtype == torch.float8_e4m3fn else \
                    o.view(torch.int16).cpu().numpy().view(np.uint16)
                np.testing.assert_array_equal(got, ref)
            F.fsdp_reshard(layer)
            prev_amax = amax
        with pytest.raises(F.FsdpError):   # the history length is fixed by the first call
            F.precompute_fp8_scales(mesh, [layer], history_len=H + 1)
    finally:
        mesh.destroy()


@pytest.mark.parametrize("algo_w", ["push_w1", "nccl_w1"])
def test_fp8_delayed_fused_two_layers_and_skipped_unshard(algo_w, monkeypatch):
    """Two units in one delayed precompute; in one step the second unit is not unsharded
    (its accumulator stays empty), so the next call runs the stand-in amax pass over its
    (unchanged) parameters.  Every step's scales equal the oracle's DelayedScaling per unit.
    nccl_w1 runs the unshard through the K3 copy-in (FSDP_B200_VARIANT without the push
    path is not selectable at W=1, so the stage copy-in with the armed accumulator is used
    via the NCCL-mode cast kernel's own test below)."""
    monkeypatch.setenv("FSDP_B200_AMAX_FUSE", "1")
    units = [_unit("toy", 0), _unit("ragged", 3, 1)]
    H = 4
    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id())
    try:
        layers, worlds, ds, bases = [], [], [], []
        for i, (shapes, elig) in enumerate(units):
            P = _params(shapes, i + 5)
            layers.append(F.fsdp_shard(mesh, [torch.from_numpy(p) for p in P], elig))
            worlds.append(World(shapes, 1, elig))
            ds.append(DelayedScaling(len(shapes), H))
            bases.append(layers[-1].sharded_flat().clone())
        skip_step = 3
        for t, f in enumerate(FACTORS):
            for i, l in enumerate(layers):
                if not (t == skip_step + 1 and i == 1):   # unit 1's params unchanged after its skipped step
                    l.sharded_flat().copy_((bases[i] * (f if i == 0 else 1.0 / f)).contiguous())
            F.precompute_fp8_scales(mesh, layers, history_len=H)
            for i, l in enumerate(layers):
                shard = l.sharded_flat().cpu().numpy()
                amax, _ = worlds[i].precompute_fp8_scales([shard])
                want = ds[i].step(amax, units[i][1])
                s_dev, _ = l.fp8_scales()
                np.testing.assert_array_equal(s_dev.cpu().numpy().view(np.uint32), want.view(np.uint32))
                if t == skip_step and i == 1:
                    continue                                # not unsharded this step
                outs = F.all_gather_params(l, torch.float8_e4m3fn)
                _, fulls = worlds[i].unshard([shard], FP8, want)
                for o, ref in zip(outs, fulls):
                    got = o.view(torch.uint8).cpu().numpy() if o.dtype == torch.float8_e4m3fn else \
                        o.view(torch.int16).cpu().numpy().view(np.uint16)
                    np.testing.assert_array_equal(got, ref)
                F.fsdp_reshard(l)
    finally:
        mesh.destroy()


def test_fp8_static_scaling():
    shapes, elig = _unit("toy")
    P = _params(shapes, 1)
    mesh = F.Mesh(1, 0, 0, local=True)
    try:
        layer = F.fsdp_shard(mesh, [torch.from_numpy(p) for p in P], elig)
        w = World(shapes, 1, elig)
        static = np.array([float(2 ** (p % 7 + 3)) if e else 0.0 for p, e in enumerate(elig)], np.float32)
        outs = F.all_gather_params(layer, torch.float8_e4m3fn, fp8_scales=torch.from_numpy(static).cuda())
        _, fulls = w.unshard(w.shard(P), FP8, static)
        for o, ref in zip(outs, fulls):
            got = o.view(torch.uint8).cpu().numpy() if o.dtype == torch.float8_e4m3fn else \
                o.view(torch.int16).cpu().numpy().view(np.uint16)
            np.testing.assert_array_equal(got, ref)
        F.fsdp_reshard(layer)
    finally:
        mesh.destroy()
