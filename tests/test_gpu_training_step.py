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
