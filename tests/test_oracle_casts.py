"""Pins for oracle/casts.py — CPU only.

bf16 and e4m3fn encoders are checked against torch CPU's casts (library routines) on
several million fp32 bit patterns spanning every exponent, plus fixed examples; the
e4m3 table/scale against SPEC worked examples and enumeration invariants."""
import json
import os

import numpy as np
import pytest
import torch

import synth
from oracle import (bf16_rne_bits, bf16_bits_to_f32, e4m3_table, e4m3_decode, e4m3_encode,
                    E4M3_MAX, fp8_scale_from_amax)
from oracle.casts import e4m3_from_fp32_scaled
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SPEC = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))


def _bits(u):
    return np.array(u, dtype=np.uint32).view(np.float32)


def _sample_patterns(n, seed):
    """Random finite fp32 bit patterns + a sweep of every exponent with edge mantissas."""
    rng = np.random.default_rng(seed)
    r = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    exps = np.arange(0, 255, dtype=np.uint32) << 23
    mants = np.array([0, 1, 0x7FFF, 0x8000, 0x8001, 0xFFFF, 0x10000, 0x18000, 0x7FFFFF,
                      0x7F8000, 0x7F7FFF, 0x400000, 0x0C0000, 0x080000, 0x040000], dtype=np.uint32)
    sweep = (exps[:, None] | mants[None, :]).reshape(-1)
    allp = np.concatenate([r, sweep, sweep | 0x80000000])
    f = allp.view(np.float32)
    return f[np.isfinite(f)]


def test_bf16_fixed_examples():
    cases = {0x3F808000: 0x3F80, 0x3F818000: 0x3F82, 0x3F808001: 0x3F81, 0x7F7FFFFF: 0x7F80,
             0xFF7FFFFF: 0xFF80, 0x00000000: 0x0000, 0x80000000: 0x8000, 0x7F7F7FFF: 0x7F7F,
             0x7F7F8000: 0x7F80}
    for u, want in cases.items():
        assert int(bf16_rne_bits(_bits([u]))[0]) == want, hex(u)
    assert int(bf16_rne_bits(np.array([1e-40], np.float32))[0]) == 0x0001  # subnormal kept


@pytest.mark.parametrize("seed", [0, 1])
def test_bf16_vs_torch_cpu(seed):
    x = np.concatenate([_sample_patterns(3_000_000, seed), synth.edge_values(200_000, seed)])
    ours = bf16_rne_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(ours, ref)


def test_bf16_widen_roundtrip():
    b = np.arange(0, 1 << 16, dtype=np.uint32).astype(np.uint16)
    f = bf16_bits_to_f32(b)
    fin = np.isfinite(f)
    np.testing.assert_array_equal(bf16_rne_bits(f[fin]), b[fin])


def test_e4m3_enumeration():
    t = e4m3_table()
    assert E4M3_MAX == SPEC["e4m3_max"]["value"]
    assert np.all(np.diff(t) > 0)                 # codes are monotone in magnitude
    assert t[1] == 2.0 ** -9                       # smallest subnormal
    assert t[0x08] == 2.0 ** -6                    # smallest normal
    assert len(t) == 127


def test_e4m3_fixed_points_all_codes():
    codes = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], dtype=np.uint8)
    vals = e4m3_decode(codes).astype(np.float32)
    np.testing.assert_array_equal(e4m3_encode(vals), codes)
    ref = torch.from_numpy(vals).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    np.testing.assert_array_equal(ref, codes)


def test_e4m3_fixed_examples():
    enc = lambda v: int(e4m3_encode(np.array([v], np.float32))[0])
    assert enc(-0.0) == 0x80
    assert enc(2.0 ** -10) == 0x00          # tie -> even (0)
    assert enc(1.5 * 2.0 ** -10) == 0x01    # 0.75 * 2^-9 -> nearest code 2^-9
    assert enc(-(2.0 ** -11)) == 0x80       # tiny negative keeps its sign
    assert enc(448.0) == 0x7E
    assert enc(464.0) == 0x7E               # clamped before rounding
    assert enc(1e30) == 0x7E and enc(-1e30) == 0xFE
    assert enc(np.inf) == 0x7E              # clamp of +inf (x*s overflow)


@pytest.mark.parametrize("seed", [0, 1])
def test_e4m3_vs_torch_cpu(seed):
    x = np.concatenate([_sample_patterns(1_500_000, seed), synth.edge_values(200_000, seed)])
    ours = e4m3_encode(x)
    ref = torch.from_numpy(x).clamp(-448.0, 448.0).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    np.testing.assert_array_equal(ours, ref)


def test_e4m3_scaled_cast_vs_torch_cpu():
    rng = np.random.default_rng(3)
    x = rng.standard_normal(500_000).astype(np.float32) * np.float32(0.02)
    for s in (np.float32(1.0), np.float32(112.0), np.float32(448.0 / 0.0731), np.float32(3.0e5)):
        ours = e4m3_from_fp32_scaled(x, s)
        y = torch.from_numpy(x) * torch.tensor(s, dtype=torch.float32)
        ref = y.clamp(-448.0, 448.0).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
        np.testing.assert_array_equal(ours, ref)


def test_e4m3_error_bound_normal_range():
    rng = np.random.default_rng(4)
    x = np.exp2(rng.uniform(-6, np.log2(448.0), 200_000)).astype(np.float32)
    q = e4m3_decode(e4m3_encode(x))
    rel = np.abs(q - x.astype(np.float64)) / x.astype(np.float64)
    assert rel.max() <= 2.0 ** -4 + 1e-12      # half an ulp of a 3-bit mantissa


def test_fp8_scale():
    ex = SPEC["fp8_dynamic_scale"]
    assert fp8_scale_from_amax(np.float32(ex["amax"])) == np.float32(ex["scale"])
    assert fp8_scale_from_amax(np.float32(0.0)) == np.float32(448.0 / np.float64(np.float32(1e-12)))
    with pytest.raises(FloatingPointError):
        fp8_scale_from_amax(np.float32(np.inf))
    with pytest.raises(FloatingPointError):
        fp8_scale_from_amax(np.float32(np.nan))


def test_nan_outside_domain():
    with pytest.raises(ValueError):
        bf16_rne_bits(np.array([np.nan], np.float32))
    with pytest.raises(ValueError):
        e4m3_encode(np.array([np.nan], np.float32))


# ----------------------------------------------------------------------------- delayed scaling (f4)
def test_delayed_scaling_worked_example():
    from oracle.scaling import DelayedScaling
    ex = json.load(open(os.path.join(GOLDEN, "fp8_delayed_scaling.json")))
    d = DelayedScaling(1, ex["history_len"])
    got = [float(d.step(np.array([a], np.float32), [True])[0]) for a in ex["amax"]]
    assert got == ex["scale"]


def test_delayed_scaling_properties():
    from oracle.scaling import DelayedScaling
    rng = np.random.default_rng(0)
    # constant amax -> constant scale equal to the dynamic one
    d = DelayedScaling(2, 16)
    for _ in range(20):
        s = d.step(np.array([3.0, 0.7], np.float32), [True, True])
        np.testing.assert_array_equal(s, fp8_scale_from_amax(np.array([3.0, 0.7], np.float32)))
    # history length 1: the scale lags the amax by exactly one step
    d = DelayedScaling(1, 1)
    a = rng.uniform(0.1, 10, 30).astype(np.float32)
    s = [d.step(a[i:i + 1], [True])[0] for i in range(30)]
    assert s[0] == fp8_scale_from_amax(a[0])
    for i in range(1, 30):
        assert s[i] == fp8_scale_from_amax(a[i - 1])
    # non-eligible params get no scale
    d = DelayedScaling(2, 4)
    assert d.step(np.array([1.0, 1.0], np.float32), [True, False])[1] == 0.0
