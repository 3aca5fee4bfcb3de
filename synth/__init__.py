"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no sharding, no casts, no reductions):
it only names parameter shapes of the paper's workloads and draws seeded random
numbers.  Both the CPU oracle (``oracle/``) and the CUDA path consume what it returns;
neither imports the other.

Workload shapes
---------------
The paper trains Llama 3.1 8B / 70B / 405B (Tables 1-4 at
PAPER.md:199-259) and wraps every ``TransformerBlock`` plus the root module in
``fully_shard``.  It does not print the model dimensions; the
public Llama 3.1 configs are used (dim / n_kv*head_dim / ffn / vocab):

* 8B : 4096 / 1024 / 14336 / 128256, 32 blocks
* 70B: 8192 / 1024 / 28672 / 128256, 80 blocks
* toy: 256 / 256 / 768 / 256, 2 blocks (BASELINE.json configs[0], "~2M params";
  1,836,288 params)

Parameters of a unit are listed in FSDP registration (FQN) order,
shapes are ``nn.Linear`` ``(out, in)``.

Value recipe
---------------------------------------
* params: fp32 ``N(0, sigma_p)``, ``sigma_p = 0.02 * 10**U(-1, 1)`` drawn per param, so
  the per-tensor amaxes differ (fp8 tensorwise scaling).
* grads: bf16 bit patterns obtained by TRUNCATING an fp32 ``N(0, 1e-3 * 10**U(-1,1))``
  draw to its top 16 bits (a generator choice, not the method's RNE cast).
* dyadic grads: ``k * 2**-10`` with ``|k| < 2**8`` (exact in bf16; every partial sum of
  pre-divided values is exact in fp32 for W = 2**j, so any reduction order is bit-exact).
* edge values: +-0, fp32 subnormals, bf16 ties, e4m3 midpoints, FLT_MAX, ...
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 241006511  # arXiv id, SURVEY.md §8 c10

KIND_PARAM = 0
KIND_GRAD = 1
KIND_EDGE = 2


# --------------------------------------------------------------------------- shapes
def llama_block(dim: int, kv: int, ffn: int):
    """One TransformerBlock's params in registration order: (fqn, shape, fp8_eligible).

    fp8 eligibility = the block's linear weights ("applied selectively to
    linear layers"); norms stay bf16."""
    return [
        ("attention.wq.weight", (dim, dim), True),
        ("attention.wk.weight", (kv, dim), True),
        ("attention.wv.weight", (kv, dim), True),
        ("attention.wo.weight", (dim, dim), True),
        ("feed_forward.w1.weight", (ffn, dim), True),
        ("feed_forward.w2.weight", (dim, ffn), True),
        ("feed_forward.w3.weight", (ffn, dim), True),
        ("attention_norm.weight", (dim,), False),
        ("ffn_norm.weight", (dim,), False),
    ]


def llama_root(dim: int, vocab: int):
    """The root FSDP unit (embedding, final norm, output projection): never fp8."""
    return [
        ("tok_embeddings.weight", (vocab, dim), False),
        ("norm.weight", (dim,), False),
        ("output.weight", (vocab, dim), False),
    ]


MODELS = {
    "toy": dict(dim=256, kv=256, ffn=768, vocab=256, n_layers=2),
    "llama3.1-8b": dict(dim=4096, kv=1024, ffn=14336, vocab=128256, n_layers=32),
    "llama3.1-70b": dict(dim=8192, kv=1024, ffn=28672, vocab=128256, n_layers=80),
}


def model_units(name: str, include_root: bool = True):
    """List of FSDP units, each a list of (fqn, shape, fp8_eligible)."""
    m = MODELS[name]
    units = [llama_block(m["dim"], m["kv"], m["ffn"]) for _ in range(m["n_layers"])]
    if include_root:
        units.append(llama_root(m["dim"], m["vocab"]))
    return units


def ragged_unit(seed: int, n_params: int | None = None, max_numel: int = 1 << 14,
                world_size: int = 8):
    """A small unit with ragged shapes: dim0 not divisible by W, dim0 < W, 1-D and 3-D
    params, numel not a multiple of 8 (misaligned copy-out / chunk-cat phases)."""
    rng = np.random.default_rng(np.random.SeedSequence([SEED_BASE, 7, seed]))
    if n_params is None:
        n_params = int(rng.integers(2, 12))
    rests = [1, 3, 5, 17, 255, 64, 129]
    out = []
    for p in range(n_params):
        kind = int(rng.integers(0, 4))
        if kind == 0:   # dim0 < W
            d0 = int(rng.integers(0, max(1, world_size)))
            shape = (d0, int(rng.choice(rests)))
        elif kind == 1:  # 1-D
            shape = (int(rng.integers(1, max_numel)),)
        elif kind == 2:  # 3-D
            shape = (int(rng.integers(1, 40)), int(rng.choice([1, 3, 7])), int(rng.choice([2, 5, 16])))
        else:
            rest = int(rng.choice(rests))
            shape = (int(rng.integers(1, max(2, max_numel // rest))), rest)
        out.append((f"p{p}", shape, bool(rng.integers(0, 2))))
    # guarantee at least one fp8-eligible and one empty-shard param
    out[0] = (out[0][0], out[0][1], True)
    return out


def sweep_unit(total_bytes: int, world_size: int):
    """Ragged unit whose bf16 all-gather output is ~total_bytes."""
    log2 = int(round(np.log2(total_bytes)))
    rng = np.random.default_rng(np.random.SeedSequence([SEED_BASE, log2, world_size]))
    n_params = int(rng.integers(2, 13))
    rests = [1, 3, 17, 255, 4096, 4099, 14336]
    target_elems = total_bytes // 2
    shapes = []
    for p in range(n_params):
        rest = int(rng.choice(rests))
        share = target_elems / n_params
        d0 = max(1, int(share // rest))
        if p % 2 == 0:
            d0 = (d0 // 8) * 8 + int(rng.integers(1, 8))
        shapes.append([d0, rest])
    shapes[0][0] = int(rng.integers(0, world_size))  # one param with d0 < W
    used = sum(d * r for d, r in shapes[:-1])
    last_rest = shapes[-1][1]
    shapes[-1][0] = max(1, (target_elems - used) // last_rest)
    return [(f"s{p}", tuple(s) if s[1] > 1 else (s[0],), bool(p % 3 != 2))
            for p, s in enumerate(shapes)]


# ---------------------------------------------------------------------------- values
def _rng(*key):
    return np.random.default_rng(np.random.SeedSequence([SEED_BASE, *[int(k) for k in key]]))


def param_values(unit: int, p: int, shape) -> np.ndarray:
    """fp32 master value of param p of unit `unit` (full, unsharded)."""
    rng = _rng(unit, p, KIND_PARAM)
    sigma = 0.02 * 10.0 ** rng.uniform(-1.0, 1.0)
    return (rng.standard_normal(size=shape, dtype=np.float32) * np.float32(sigma)).astype(np.float32)


def grad_bf16_bits(unit: int, p: int, rank: int, shape) -> np.ndarray:
    """Rank `rank`'s full bf16 gradient of param p as uint16 bit patterns (truncated draw)."""
    rng = _rng(unit, p, KIND_GRAD, rank)
    sigma = 1e-3 * 10.0 ** rng.uniform(-1.0, 1.0)
    g = rng.standard_normal(size=shape, dtype=np.float32) * np.float32(sigma)
    return (g.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def grad_fp32(unit: int, p: int, rank: int, shape) -> np.ndarray:
    rng = _rng(unit, p, KIND_GRAD, rank, 32)
    sigma = 1e-3 * 10.0 ** rng.uniform(-1.0, 1.0)
    return (rng.standard_normal(size=shape, dtype=np.float32) * np.float32(sigma)).astype(np.float32)


def dyadic_grad_bf16_bits(unit: int, p: int, rank: int, shape) -> np.ndarray:
    """k * 2**-10, |k| < 2**8, as exact bf16 bit patterns."""
    rng = _rng(unit, p, KIND_GRAD, rank, 2)
    k = rng.integers(-(1 << 8) + 1, 1 << 8, size=shape)
    v = np.ldexp(k.astype(np.float32), -10).astype(np.float32)
    return (v.view(np.uint32) >> 16).astype(np.uint16)


def edge_values(n: int, seed: int = 0) -> np.ndarray:
    """fp32 values concentrated on rounding boundaries (all finite)."""
    rng = _rng(seed, KIND_EDGE)
    pools = []
    # +-0, smallest/largest subnormal and normal, FLT_MAX
    specials = np.array([0x00000000, 0x80000000, 0x00000001, 0x80000001, 0x007FFFFF,
                         0x00800000, 0x7F7FFFFF, 0xFF7FFFFF, 0x3F800000, 0xBF800000,
                         0x3F808000, 0x3F818000, 0x3F80C000, 0x7F7F8000, 0x7F7F7FFF],
                        dtype=np.uint32)
    pools.append(specials.view(np.float32))
    # bf16 ties and near-ties: low 16 bits 0x8000 +- small
    hi = rng.integers(0, 0x7F7F, size=n // 4, dtype=np.uint32)
    lo = rng.choice(np.array([0x7FFF, 0x8000, 0x8001, 0x0000, 0xFFFF], dtype=np.uint32), size=n // 4)
    sign = rng.integers(0, 2, size=n // 4, dtype=np.uint32) << 31
    pools.append(((hi << 16) | lo | sign).view(np.float32))
    # e4m3 grid midpoints and their fp32 neighbours in [2^-10, 480]
    e = rng.integers(-10, 9, size=n // 4)
    m = rng.integers(0, 16, size=n // 4)  # odd m/16 = midpoint between two e4m3 codes
    mid = np.ldexp(1.0 + m / 16.0, e).astype(np.float32)
    bump = rng.integers(-1, 2, size=n // 4).astype(np.int32)
    mid = (mid.view(np.int32) + bump).view(np.float32)
    mid = mid * np.where(rng.integers(0, 2, size=n // 4) == 0, np.float32(1), np.float32(-1))
    pools.append(mid.astype(np.float32))
    # random finite bit patterns
    r = rng.integers(0, 1 << 32, size=max(0, n - sum(len(x) for x in pools)), dtype=np.uint64).astype(np.uint32)
    rf = r.view(np.float32)
    rf = np.where(np.isfinite(rf), rf, np.float32(1.0))
    pools.append(rf.astype(np.float32))
    out = np.concatenate(pools).astype(np.float32)
    return out[:n]
