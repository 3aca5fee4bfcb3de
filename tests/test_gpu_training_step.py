"""Training steps through the library vs a single-device run, W=1 on one GPU:
bf16 unshard -> forward/backward -> fp32 reduce-scatter -> SGD on the fp32 shards equals the
single-device mixed-precision run bit for bit (same kernels, same order).  Multi-GPU
versions (W=2/4, P2P and NCCL) run in tests/mgpu_worker.py."""
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F

import toy_train  # noqa: E402


@pytest.mark.parametrize("local", [False, True])
def test_training_steps_match_single_device(local):
    mesh = F.Mesh(1, 0, 0, local=True) if local else F.Mesh(1, 0, 0, unique_id=F.get_unique_id())
    try:
        ref = toy_train.reference_steps(4, 1)
        got, metas = toy_train.fsdp_steps(F, mesh, 0, 4)
        toy_train.compare(ref, got, metas, exact=True)
    finally:
        mesh.destroy()


def test_sharded_state_dict_roundtrip():
    """the sharded state is the per-rank shards + Shard(0) placement, no
    communication; concatenating every rank's rows reproduces the full parameters, and a
    save/load round trip restores the shard bit for bit."""
    import numpy as np
    from test_gpu_parity import _unit, _params, Emu
    shapes, elig = _unit("ragged", 2, 3)
    P = _params(shapes, 2)
    emu = Emu(shapes, elig, 3, P)
    try:
        states = [l.sharded_state_dict() for l in emu.layers]
        for p, full in enumerate(P):
            rows = [s[f"p{p}"]["local"].cpu().numpy() for s in states]
            begins = [s[f"p{p}"]["row_begin"] for s in states]
            assert begins == sorted(begins)
            np.testing.assert_array_equal(np.concatenate(rows).reshape(full.shape), full)
        saved = {k: {**v, "local": v["local"].cpu().clone()} for k, v in states[1].items()}
        emu.layers[1].sharded_flat().zero_()
        emu.layers[1].load_sharded_state_dict(saved)
        for p in range(len(shapes)):
            assert torch.equal(emu.layers[1].sharded_param(p).cpu(), saved[f"p{p}"]["local"])
        with pytest.raises(ValueError):
            emu.layers[0].load_sharded_state_dict(saved)    # another rank's placement
    finally:
        emu.close()
