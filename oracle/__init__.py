"""CPU oracle for the FSDP2 per-parameter Shard(0) step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2410_06511_b200``) never imports, calls or links it, and the two share no
code: only the seeded input generators in ``synth/`` serve both.

What it computes (PAPER.md = /root/reference/PAPER.md):

* sharding metadata and initial shards  — PAPER.md:460 (``appendix:fsdp``: "parameters
  are now represented as DTensors sharded on the tensor dimension 0")       [layout.py]
* unshard = copy-in (bf16, or float8 e4m3 with per-tensor scale) -> all-gather ->
  copy-out — PAPER.md:154, :157, :417, :464                                  [world.py]
* fp8 amax / scale precompute — PAPER.md:157 (per-tensor dynamic scaling)   [world.py]
* gradient reduce-scatter in fp32 with a single pre-division by W —
  PAPER.md:154, :417, :466, :544                                             [world.py]
* the two casts (fp32 -> bf16 RNE, fp32 -> e4m3fn RNE with clamp)           [casts.py]

Readings of silent/ambiguous passages are listed in DESIGN.md §3 and cited inline.
Representation: bf16 values are uint16 bit patterns, e4m3fn values are uint8 codes,
fp32 is float32, exact references are float64.

Pins: every function is pinned by ``tests/test_oracle_*.py`` (``-m "not gpu"``) against
closed forms, torch-CPU library casts, SPEC worked examples (tests/golden/) and
brute force.  Parity-unpinned parts: none for integer/byte work; for the fp32
reduce-scatter of non-dyadic data only the error bound is pinned (DESIGN.md §3 R10) — and
that bound itself (``rs_error_ok``) is pinned from both sides, as is the bf16-reduce
branch of ``rs_copy_in`` (rounding after the single division; exact rational arithmetic),
in tests/test_oracle_pins_r2.py.
"""
from .layout import ParamMeta, UnitLayout, unit_layout, round_up, ALIGN_ELEMS, ALIGN_BYTES
from .casts import (bf16_rne_bits, bf16_bits_to_f32, e4m3_table, e4m3_decode,
                    e4m3_encode, E4M3_MAX, fp8_scale_from_amax, AMAX_EPS)
from .world import World, HsdpWorld

__all__ = [
    "ParamMeta", "UnitLayout", "unit_layout", "round_up", "ALIGN_ELEMS", "ALIGN_BYTES",
    "bf16_rne_bits", "bf16_bits_to_f32", "e4m3_table", "e4m3_decode", "e4m3_encode",
    "E4M3_MAX", "fp8_scale_from_amax", "AMAX_EPS", "World", "HsdpWorld",
]
