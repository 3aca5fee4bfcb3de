"""Element casts used by unshard — oracle (test infrastructure only).

* fp32 -> bf16, round to nearest, ties to even ("we use torch.bfloat16 on
  parameters all-gather").  Written as the definition: of the two bf16
  neighbours of |x| (the truncation and the next value up) take the nearer, on a tie the
  one with an even bf16 mantissa; magnitudes past the largest finite bf16 by at least half
  an ulp round to infinity (IEEE RNE overflow).  NaN inputs are outside the domain
  (reading R5) and raise.
* fp32 -> float8 e4m3fn given a per-tensor scale ("per-tensor scaling ...
  Float8 all-gather"): ``y = fp32(x * s)`` (one IEEE fp32 multiply), clamp to
  ``[-E4M3_MAX, E4M3_MAX]``, then the nearest of the 127 finite e4m3fn magnitudes, ties to
  the code with even LSB, sign bit of y kept (reading R4/R7).
* scale from amax (reading R7): ``s = fp32(E4M3_MAX / fp64(max(amax, 1e-12)))``,
  SPEC.md:417 "scale = E4M3_MAX / amax", "amax == 0 -> scale clamped".
"""
from __future__ import annotations

import numpy as np

_CHUNK = 1 << 22


# ----------------------------------------------------------------------------- bf16
def _bf16_rne_chunk(x: np.ndarray) -> np.ndarray:
    u = x.view(np.uint32).astype(np.uint64)
    sign = u & 0x80000000
    mag = u & 0x7FFFFFFF
    if np.any(mag > 0x7F800000):
        raise ValueError("NaN input to the bf16 cast (outside the oracle's domain, reading R5)")
    lo = mag & 0xFFFF0000                      # truncated bf16 neighbour (as fp32 bits)
    hi = lo + 0x10000                          # next bf16 value up in magnitude
    val_x = np.abs(x.astype(np.float64))
    val_lo = lo.astype(np.uint32).view(np.float32).astype(np.float64)
    # bits 0x7F800000 as the "next value up" stand for 2**128 (IEEE overflow threshold)
    val_hi = np.where(hi >= 0x7F800000, np.float64(2.0 ** 128),
                      np.minimum(hi, 0x7F7FFFFF).astype(np.uint32).view(np.float32).astype(np.float64))
    d_lo = val_x - val_lo                      # exact in fp64
    d_hi = val_hi - val_x
    lo_even = ((lo >> 16) & 1) == 0
    take_hi = (d_hi < d_lo) | ((d_hi == d_lo) & ~lo_even)
    chosen = np.where(take_hi, hi, lo)
    chosen = np.where(mag == 0x7F800000, mag, chosen)   # +-inf stays inf
    return ((sign | chosen) >> 16).astype(np.uint16)


def bf16_rne_bits(x: np.ndarray) -> np.ndarray:
    """fp32 array -> bf16 bit patterns (uint16), RNE."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    out = np.empty(x.size, dtype=np.uint16)
    for s in range(0, x.size, _CHUNK):
        out[s:s + _CHUNK] = _bf16_rne_chunk(x[s:s + _CHUNK])
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> fp32 values (exact widening)."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ----------------------------------------------------------------------------- e4m3fn
def e4m3_table() -> np.ndarray:
    """Magnitudes of the 127 finite non-negative e4m3fn codes 0x00..0x7E (fp64).

    e4m3fn: 1 sign, 4 exponent (bias 7), 3 mantissa bits; exponent field 0 is subnormal
    (m/8 * 2**-6); code 0x7F (and 0xFF) is NaN, there are no infinities."""
    codes = np.arange(0x7F)
    e = (codes >> 3) & 0xF
    m = codes & 0x7
    sub = m.astype(np.float64) / 8.0 * 2.0 ** -6
    nrm = (1.0 + m.astype(np.float64) / 8.0) * np.power(2.0, (e - 7).astype(np.float64))
    return np.where(e == 0, sub, nrm)


_TABLE = e4m3_table()
E4M3_MAX = float(_TABLE.max())          # 448 by enumeration
AMAX_EPS = np.float32(1e-12)            # reading R7


def e4m3_decode(codes: np.ndarray) -> np.ndarray:
    c = np.asarray(codes, dtype=np.uint8)
    mag_code = (c & 0x7F).astype(np.int64)
    v = np.where(mag_code == 0x7F, np.nan, _TABLE[np.minimum(mag_code, 0x7E)])
    return np.where((c & 0x80) != 0, -v, v)


def _e4m3_encode_chunk(y: np.ndarray) -> np.ndarray:
    if np.any(np.isnan(y)):
        raise ValueError("NaN input to the e4m3 cast (outside the oracle's domain, reading R5)")
    neg = np.signbit(y)
    a = np.minimum(np.abs(y.astype(np.float64)), E4M3_MAX)   # the clamp (reading R4)
    idx = np.searchsorted(_TABLE, a, side="left")             # _TABLE[idx-1] < a <= _TABLE[idx]
    hi = np.minimum(idx, 0x7E)
    lo = np.maximum(idx - 1, 0)
    d_lo = a - _TABLE[lo]
    d_hi = _TABLE[hi] - a
    take_hi = (d_hi < d_lo) | ((d_hi == d_lo) & ((lo & 1) == 1))
    code = np.where(take_hi, hi, lo).astype(np.uint8)
    return np.where(neg, code | np.uint8(0x80), code).astype(np.uint8)


def e4m3_encode(y: np.ndarray) -> np.ndarray:
    """Already-scaled fp32 values -> e4m3fn codes (clamp + nearest, ties to even)."""
    y = np.ascontiguousarray(y, dtype=np.float32).reshape(-1)
    out = np.empty(y.size, dtype=np.uint8)
    for s in range(0, y.size, _CHUNK):
        out[s:s + _CHUNK] = _e4m3_encode_chunk(y[s:s + _CHUNK])
    return out


def e4m3_from_fp32_scaled(x: np.ndarray, scale: np.float32) -> np.ndarray:
    """The fp8 copy-in cast: y = fp32(x * s) (IEEE fp32 multiply), then e4m3_encode."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    with np.errstate(over="ignore"):
        y = (x * np.float32(scale)).astype(np.float32)
    return e4m3_encode(y)


def fp8_scale_from_amax(amax) -> np.ndarray:
    """s = fp32(E4M3_MAX / fp64(max(amax, EPS))) elementwise (reading R7)."""
    a = np.asarray(amax, dtype=np.float32)
    if not np.all(np.isfinite(a)):
        raise FloatingPointError("non-finite amax (SPEC.md:38: NaN/Inf is an error surfaced)")
    a = np.maximum(a, AMAX_EPS)
    return (np.float64(E4M3_MAX) / a.astype(np.float64)).astype(np.float32)
