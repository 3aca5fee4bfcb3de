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


@pytest.mark.parametrize("H", [1, 4, 16])
def test_fp8_delayed_scaling_sequence(H):
    shapes, elig = _unit("toy")
    P = _params(shapes, 0)
    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id())
    try:
        layer = F.fsdp_shard(mesh, [torch.from_numpy(p) for p in P], elig)
        w = World(shapes, 1, elig)
        d = DelayedScaling(len(shapes), H)
        base = layer.sharded_flat().clone()
        for f in [1.0, 2.0, 0.25, 8.0, 1.0, 1.0, 1.0, 0.5, 3.0]:
            cur = (base * f).contiguous()
            layer.sharded_flat().copy_(cur)
            F.precompute_fp8_scales(mesh, [layer], history_len=H)
            s_dev, a_dev = layer.fp8_scales()
            shard = cur.cpu().numpy()
            amax, _ = w.precompute_fp8_scales([shard])
            want = d.step(amax, elig)
            np.testing.assert_array_equal(a_dev.cpu().numpy().view(np.uint32), amax.view(np.uint32))
            np.testing.assert_array_equal(s_dev.cpu().numpy().view(np.uint32), want.view(np.uint32))
            outs = F.all_gather_params(layer, torch.float8_e4m3fn)
            _, fulls = w.unshard([shard], FP8, want)
            for o, ref in zip(outs, fulls):
                got = o.view(torch.uint8).cpu().numpy() if o.dtype == torch.float8_e4m3fn else \
                    o.view(torch.int16).cpu().numpy().view(np.uint16)
                np.testing.assert_array_equal(got, ref)
            F.fsdp_reshard(layer)
        with pytest.raises(F.FsdpError):   # the history length is fixed by the first call
            F.precompute_fp8_scales(mesh, [layer], history_len=H + 1)
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
