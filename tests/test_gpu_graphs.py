"""CUDA graphs (the launch-bound inner loop captured once, replayed every step): a whole FSDP
step through the library — unshard with prefetch, reshard, reduce-scatter for every unit,
optionally the fp8 scale precompute — is captured with torch.cuda.graph and replayed.
Replays must equal eager execution bit for bit, follow in-place input changes (checked
against the oracle), and capture must refuse (FSDP_ERR_STATE) a call whose buffers were
never warmed up eagerly.  The W > 1 version (P2P handshake epochs advanced on the device;
NCCL collectives inside the graph) runs in tests/mgpu_worker.py."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F

import graph_step  # noqa: E402
import synth  # noqa: E402
from oracle import World  # noqa: E402
from oracle.world import BF16, FP8  # noqa: E402


@pytest.mark.parametrize("fp8", [False, True])
def test_graph_replay_equals_eager_and_follows_inputs(fp8):
    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id())
    try:
        layers, grads, params = graph_step.setup(F, mesh)
        s = torch.cuda.Stream()
        outs = graph_step.outs_for(layers, fp8)
        with torch.cuda.stream(s):
            graph_step.step(F, mesh, layers, grads, s, outs, fp8)   # warm-up: pools, precompute tables
        s.synchronize()
        eager_g = [l.sharded_grad_flat().clone() for l in layers]
        eager_o = [[o.clone() for o in row] for row in outs]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            graph_step.step(F, mesh, layers, grads, s, outs, fp8)
        for l in layers:
            l.sharded_grad_flat().zero_()
        for row in outs:
            for o in row:
                o.zero_()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        for l, e in zip(layers, eager_g):
            assert torch.equal(l.sharded_grad_flat(), e)
        for row, erow in zip(outs, eager_o):
            for o, e in zip(row, erow):
                assert torch.equal(o, e)
        params = graph_step.refill(layers, grads, params, 0, 700)
        g.replay()
        torch.cuda.synchronize()
        for ui, l in enumerate(layers):
            shapes, elig, P2 = params[ui]
            w = World(shapes, 1, elig)
            sh = w.shard(P2)
            if fp8:
                _, scale = w.precompute_fp8_scales(sh)
                _, fulls = w.unshard(sh, FP8, scale)
            else:
                _, fulls = w.unshard(sh, BF16)
            for o, want in zip(outs[ui], fulls):
                got = o.cpu().numpy() if o.dtype == torch.uint8 else o.view(torch.int16).cpu().numpy().view(np.uint16)
                np.testing.assert_array_equal(got, want)
            G = [[synth.grad_bf16_bits(ui + 700, p, 0, s_) for p, s_ in enumerate(shapes)]]
            ref = w.reduce_scatter_grads(G, BF16, True)[0]
            for p in range(l.P):
                np.testing.assert_array_equal(l.sharded_grad(p).cpu().numpy(), ref["order"][p])
        # eager calls after replays (pool buffers released inside the capture) give the same result
        after_g = [l.sharded_grad_flat().clone() for l in layers]
        with torch.cuda.stream(s):
            graph_step.step(F, mesh, layers, grads, s, outs, fp8)
        s.synchronize()
        for l, e in zip(layers, after_g):
            assert torch.equal(l.sharded_grad_flat(), e)
        del g
    finally:
        torch.cuda.synchronize()
        mesh.destroy()


def test_capture_without_warmup_is_a_state_error():
    mesh = F.Mesh(1, 0, 0, unique_id=F.get_unique_id())
    try:
        layers, grads, _ = graph_step.setup(F, mesh)
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with pytest.raises(F.FsdpError) as e:
            with torch.cuda.graph(g, stream=s):
                F.fsdp_unshard(layers[0], stream=s)      # no eager unshard ever allocated a buffer
        assert e.value.status_name == "FSDP_ERR_STATE"
        assert "eagerly" in str(e.value)
        # the library state is unchanged: the same call works eagerly afterwards
        with torch.cuda.stream(s):
            F.all_gather_params(layers[0], stream=s)
            F.fsdp_reshard(layers[0], stream=s)
        s.synchronize()
    finally:
        torch.cuda.synchronize()
        mesh.destroy()
