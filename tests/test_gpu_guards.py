"""Guard bands for the segmented kernels (compute-sanitizer is closed on this pool).

Every output lives inside one larger sentinel-filled buffer: per-param outputs of the
copy-out kernel are placed at odd 2-byte offsets (misaligned destinations) with sentinel
gaps between them, the all-gather slot / RS input buffers get a sentinel tail.  Results
must equal the oracle and every sentinel byte must survive."""
import numpy as np
import pytest
import torch

from oracle import World
from oracle.world import BF16, FP8, FP32

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_06511_b200 as F

from test_gpu_parity import _unit, _params, Emu, KINDS  # noqa: E402

SENT = 0x5A
TAIL = 256


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", [1, 3, 8])
@pytest.mark.parametrize("fp8", [False, True])
def test_copy_out_misaligned_outputs_guarded(kind, seed, W, fp8):
    shapes, elig = _unit(kind, seed, W)
    P = _params(shapes, seed)
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, P)
    try:
        shards = w.shard(P)
        scale = w.precompute_fp8_scales(shards)[1] if fp8 else None
        ag, fulls = w.unshard(shards, FP8 if fp8 else BF16, scale)
        # outputs at 2-byte (not 16-byte) aligned offsets with 50-byte sentinel gaps
        offs, pos = [], 2
        for f in fulls:
            offs.append(pos)
            pos += f.size * f.itemsize + 50
        big = torch.full((pos + TAIL,), SENT, dtype=torch.uint8, device="cuda")
        outs = [big[o:o + f.size * f.itemsize] for o, f in zip(offs, fulls)]
        F.stage_copy_out(emu.layers[W - 1], torch.float8_e4m3fn if fp8 else torch.bfloat16,
                         torch.from_numpy(ag).cuda(), outs)
        torch.cuda.synchronize()
        b = big.cpu().numpy()
        written = np.zeros(b.size, dtype=bool)
        for o, f in zip(offs, fulls):
            n = f.size * f.itemsize
            np.testing.assert_array_equal(b[o:o + n].view(f.dtype).reshape(f.shape), f)
            written[o:o + n] = True
        assert np.all(b[~written] == SENT)
    finally:
        emu.close()


@pytest.mark.parametrize("kind,seed", KINDS)
@pytest.mark.parametrize("W", [1, 3, 8])
def test_copy_in_and_rs_copy_in_tails_guarded(kind, seed, W):
    shapes, elig = _unit(kind, seed, W)
    P = _params(shapes, seed)
    w = World(shapes, W, elig)
    emu = Emu(shapes, elig, W, P)
    try:
        shards = w.shard(P)
        l = emu.layers[W - 1]
        for fp8 in (False, True):
            n = l.S_bytes_fp8 if fp8 else 2 * l.S
            buf = torch.full((n + TAIL,), SENT, dtype=torch.uint8, device="cuda")
            scale = w.precompute_fp8_scales(shards)[1] if fp8 else None
            F.stage_copy_in(l, torch.float8_e4m3fn if fp8 else torch.bfloat16, buf,
                            fp8_scales=torch.from_numpy(scale).cuda() if fp8 else None)
            torch.cuda.synchronize()
            b = buf.cpu().numpy()
            np.testing.assert_array_equal(b[:n], w.copy_in(shards[W - 1], FP8 if fp8 else BF16, scale))
            assert np.all(b[n:] == SENT)
        import synth
        g = [synth.grad_bf16_bits(seed, p, 0, s) for p, s in enumerate(shapes)]
        gt = [torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) for x in g]
        n = 4 * W * l.S
        buf = torch.full((n + TAIL,), SENT, dtype=torch.uint8, device="cuda")
        F.stage_rs_copy_in(l, gt, torch.float32, True, buf)
        torch.cuda.synchronize()
        b = buf.cpu().numpy()
        np.testing.assert_array_equal(b[:n].view(np.float32), w.rs_copy_in(g, BF16, True, FP32))
        assert np.all(b[n:] == SENT)
    finally:
        emu.close()
