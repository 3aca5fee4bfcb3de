"""Shard(0) metadata of one FSDP unit — oracle (test infrastructure only).

Definition (appendix:fsdp: every parameter is a DTensor sharded on dim 0
over the data-parallel mesh; the default mesh is all ranks):

* ``c_p = ceil(d0_p / W)`` rows per chunk (reading R1: ceiling division with trailing
  empty chunks, "chunk c covers rows [c*ceil(n/W), min((c+1)*ceil(n/W), n))")
* rank r owns rows ``[b, e)`` with ``b = min(r*c_p, d0_p)``, ``e = min((r+1)*c_p, d0_p)``
* padded shard numel ``n_p = c_p * rest_p`` (rest_p = product of the other dims);
  rows ``[e-b, c_p)`` of the shard are zero padding (reading R1)
* flat layout (reading R2): ``off_p = sum_{q<p} round_up(n_q, 16)`` elements,
  ``S = sum_p round_up(n_p, 16)``.  Param order = caller order (reading R3).
* mixed float8 all-gather buffer (reading R6/R8): param p occupies
  ``round_up(n_p * e_p, 16)`` bytes at ``boff_p`` where ``e_p`` = 1 (e4m3) for fp8-eligible
  params and 2 (bf16) otherwise.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

ALIGN_ELEMS = 16   # reading R2
ALIGN_BYTES = 16   # reading R2 for the mixed fp8/bf16 byte buffer


def round_up(n: int, a: int) -> int:
    return ((n + a - 1) // a) * a


def ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


@dataclass(frozen=True)
class ParamMeta:
    shape: Tuple[int, ...]
    dim0: int
    rest: int
    chunk_rows: int      # c_p
    row_begin: int       # b
    row_count: int       # e - b (0 for trailing empty shards)
    padded_numel: int    # n_p
    elem_offset: int     # off_p in the fp32 shard / bf16 all-gather / fp32 RS layouts
    fp8_eligible: bool
    byte_offset_fp8: int  # boff_p in the mixed fp8 all-gather byte layout

    @property
    def numel(self) -> int:
        return self.dim0 * self.rest


@dataclass(frozen=True)
class UnitLayout:
    world_size: int
    rank: int
    params: List[ParamMeta] = field(default_factory=list)
    S: int = 0            # per-rank flat length in elements
    S_bytes_fp8: int = 0  # per-rank byte length of the mixed fp8 all-gather slot


def unit_layout(shapes: Sequence[Sequence[int]], world_size: int, rank: int,
                fp8_eligible: Sequence[bool] | None = None) -> UnitLayout:
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("invalid world_size/rank")
    if fp8_eligible is None:
        fp8_eligible = [False] * len(shapes)
    metas = []
    off = 0
    boff = 0
    for shape, elig in zip(shapes, fp8_eligible):
        shape = tuple(int(s) for s in shape)
        if len(shape) == 0:
            raise ValueError("0-dim parameters cannot be Shard(0)-sharded (reading R4)")
        d0 = shape[0]
        rest = 1
        for s in shape[1:]:
            rest *= s
        c = ceil_div(d0, world_size)
        b = min(rank * c, d0)
        e = min((rank + 1) * c, d0)
        n = c * rest
        esize = 1 if elig else 2
        metas.append(ParamMeta(shape, d0, rest, c, b, e - b, n, off, bool(elig), boff))
        off += round_up(n, ALIGN_ELEMS)
        boff += round_up(n * esize, ALIGN_BYTES)
    return UnitLayout(world_size, rank, metas, off, boff)
