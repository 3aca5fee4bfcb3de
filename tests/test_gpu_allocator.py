"""fsdp_mesh_set_allocator (SURVEY.md §8(b) "Ownership": device memory from a caller-supplied
allocator, wired by the binding to the torch caching allocator): the bulk buffers are
accounted by torch, results are identical under either allocator, and a failing or
misaligned callback is an error with no side effects."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F
    from paper_2410_06511_b200 import _capi as capi

import synth  # noqa: E402
from oracle import World  # noqa: E402
from oracle.world import BF16  # noqa: E402


def _unit():
    u = synth.model_units("toy")[0]
    return [s for _, s, _ in u], [e for _, _, e in u]


def test_torch_allocator_accounts_bulk_buffers():
    shapes, elig = _unit()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(0)
    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id())
    assert mesh.allocator == "torch"
    try:
        layer = F.fsdp_shard(mesh, None, elig, shapes=shapes)
        after_shard = torch.cuda.memory_allocated(0)
        assert after_shard - base >= 2 * 4 * layer.S          # fp32 shard + sharded grad
        F.all_gather_params(layer, torch.bfloat16)            # NCCL-path pool slot (W=1)
        assert torch.cuda.memory_allocated(0) > after_shard
        F.fsdp_reshard(layer)
        layer.destroy()
    finally:
        mesh.destroy()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated(0) == base           # everything freed through torch


@pytest.mark.parametrize("allocator", ["torch", "cuda"])
def test_results_identical_under_either_allocator(allocator):
    shapes, elig = _unit()
    P = [synth.param_values(0, p, s) for p, s in enumerate(shapes)]
    w = World(shapes, 1, elig)
    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id(), allocator=allocator)
    try:
        layer = F.fsdp_shard(mesh, [torch.from_numpy(p) for p in P], elig)
        outs = F.all_gather_params(layer, torch.bfloat16)
        _, fulls = w.unshard(w.shard(P), BF16)
        for o, want in zip(outs, fulls):
            np.testing.assert_array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), want)
        F.fsdp_reshard(layer)
        G = [[synth.grad_bf16_bits(0, p, 0, s) for p, s in enumerate(shapes)]]
        gt = [torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in G[0]]
        F.reduce_scatter_grads(layer, gt)
        F.fsdp_wait_reduce_scatter(layer)
        ref = w.reduce_scatter_grads(G, BF16, True)[0]
        for p in range(len(shapes)):
            np.testing.assert_array_equal(layer.sharded_grad(p).cpu().numpy(), ref["order"][p])
    finally:
        mesh.destroy()


def _set(mesh, alloc, free):
    cbs = (capi.ALLOC_FN(alloc), capi.FREE_FN(free))
    mesh._alloc_cbs = cbs
    capi.call("fsdp_mesh_set_allocator", mesh.handle, cbs[0], cbs[1], None)


def test_failing_allocator_is_out_of_memory():
    shapes, elig = _unit()
    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id(), allocator="cuda")
    try:
        _set(mesh, lambda ctx, n, d, out: 1, lambda ctx, p, d: None)
        with pytest.raises(F.FsdpError) as e:
            F.fsdp_shard(mesh, None, elig, shapes=shapes)
        assert e.value.status_name == "FSDP_ERR_OUT_OF_MEMORY"
        assert mesh.layers == []
    finally:
        mesh.destroy()


def test_misaligned_allocator_is_rejected():
    shapes, elig = _unit()
    freed = []
    keep = []

    def alloc(ctx, n, d, out):
        t = torch.empty(int(n) + 512, dtype=torch.uint8, device="cuda")
        keep.append(t)
        out[0] = t.data_ptr() + 8                      # deliberately not 256-byte aligned
        return 0

    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id(), allocator="cuda")
    try:
        _set(mesh, alloc, lambda ctx, p, d: freed.append(p))
        with pytest.raises(F.FsdpError) as e:
            F.fsdp_shard(mesh, None, elig, shapes=shapes)
        assert e.value.status_name == "FSDP_ERR_INVALID_ARGUMENT"
        assert len(freed) == 1                          # the rejected block went back to its owner
        # both NULL restores cudaMalloc; one NULL is an argument error
        capi.call("fsdp_mesh_set_allocator", mesh.handle, capi.ALLOC_FN(), capi.FREE_FN(), None)
        layer = F.fsdp_shard(mesh, None, elig, shapes=shapes)
        layer.destroy()
        with pytest.raises(F.FsdpError):
            capi.call("fsdp_mesh_set_allocator", mesh.handle, capi.ALLOC_FN(lambda *a: 0),
                              capi.FREE_FN(), None)
    finally:
        mesh.destroy()
