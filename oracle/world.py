"""Plain CPU simulation of W ranks running the FSDP2 Shard(0) hot path — oracle
(test infrastructure only; see oracle/__init__.py).

Collectives are plain loops ("reduction performed in ascending rank order"):
* all-gather   = concatenation of the per-rank slots in rank order
* reduce-scatter = per-rank chunk sums, ascending rank order
* all-reduce(max) of the per-param local amax (SPEC.md:162 pattern)

Step order follows the paper's description of FSDP2:
unshard = copy-in (cast) -> all-gather -> copy-out into per-parameter full tensors
("multi-tensor allgather"; bf16 all-gather PAPER.md:417; Float8 all-gather
PAPER.md:157); post-backward = pre-divide the local fp32 reduce-scatter input by W once
 -> fp32 reduce-scatter -> sharded gradient.
"""
from __future__ import annotations

import math
from typing import List, Sequence

import numpy as np

from .layout import unit_layout
from .casts import (bf16_rne_bits, bf16_bits_to_f32, e4m3_from_fp32_scaled,
                    fp8_scale_from_amax)

BF16 = "bf16"
FP8 = "fp8"
FP32 = "fp32"


class World:
    """W simulated ranks holding one FSDP unit with the given parameter shapes."""

    def __init__(self, shapes: Sequence[Sequence[int]], world_size: int,
                 fp8_eligible: Sequence[bool] | None = None):
        self.shapes = [tuple(int(s) for s in sh) for sh in shapes]
        self.W = int(world_size)
        self.fp8_eligible = list(fp8_eligible) if fp8_eligible is not None else [False] * len(shapes)
        self.layouts = [unit_layout(self.shapes, self.W, r, self.fp8_eligible) for r in range(self.W)]
        self.S = self.layouts[0].S
        self.S_bytes_fp8 = self.layouts[0].S_bytes_fp8
        self.P = len(self.shapes)

    # ------------------------------------------------------------------ a1: shard
    def shard(self, full_params: Sequence[np.ndarray]) -> List[np.ndarray]:
        """Per rank: flat fp32[S]; param p's rows [b, e) at off_p, then zeros (reading R1)."""
        shards = []
        for lay in self.layouts:
            buf = np.zeros(lay.S, dtype=np.float32)
            for m, full in zip(lay.params, full_params):
                rows = np.asarray(full, dtype=np.float32).reshape(m.dim0, m.rest)[m.row_begin:m.row_begin + m.row_count]
                buf[m.elem_offset:m.elem_offset + m.row_count * m.rest] = rows.reshape(-1)
            shards.append(buf)
        return shards

    # ------------------------------------------------------- a2: fp8 amax / scales
    def local_amax(self, shard: np.ndarray) -> np.ndarray:
        """max |x| over this rank's (padded) shard of every fp8-eligible param; 0 otherwise."""
        lay = self.layouts[0]
        out = np.zeros(self.P, dtype=np.float32)
        for p, m in enumerate(lay.params):
            if m.fp8_eligible and m.padded_numel > 0:
                out[p] = np.max(np.abs(shard[m.elem_offset:m.elem_offset + m.padded_numel]))
        return out

    def precompute_fp8_scales(self, shards: Sequence[np.ndarray]):
        """amax_p = all-reduce(max) of the local amaxes; s_p from fp8_scale_from_amax.
        Returns (amax[P], scale[P]); non-eligible params get 0 for both."""
        amax = self.local_amax(shards[0])
        for r in range(1, self.W):
            amax = np.maximum(amax, self.local_amax(shards[r]))
        scale = np.zeros(self.P, dtype=np.float32)
        for p in range(self.P):
            if self.fp8_eligible[p]:
                scale[p] = fp8_scale_from_amax(amax[p])
        return amax, scale

    # ------------------------------------------------------------ a3: copy-in
    def copy_in(self, shard: np.ndarray, dtype: str = BF16, scales=None) -> np.ndarray:
        """Contents of this rank's all-gather slot, as bytes (uint8)."""
        if dtype == BF16:
            return bf16_rne_bits(shard).view(np.uint8)
        if dtype != FP8:
            raise ValueError(dtype)
        lay = self.layouts[0]
        buf = np.zeros(lay.S_bytes_fp8, dtype=np.uint8)
        for p, m in enumerate(lay.params):
            seg = shard[m.elem_offset:m.elem_offset + m.padded_numel]
            if m.fp8_eligible:
                buf[m.byte_offset_fp8:m.byte_offset_fp8 + m.padded_numel] = e4m3_from_fp32_scaled(seg, scales[p])
            else:
                b = bf16_rne_bits(seg).view(np.uint8)
                buf[m.byte_offset_fp8:m.byte_offset_fp8 + b.size] = b
        return buf

    # --------------------------------------------------------- a4: all-gather
    def all_gather(self, slots: Sequence[np.ndarray]) -> np.ndarray:
        """Rank-major concatenation, identical on every rank."""
        return np.concatenate([np.asarray(s, dtype=np.uint8) for s in slots])

    # ----------------------------------------------------------- a5: copy-out
    def copy_out(self, ag: np.ndarray, dtype: str = BF16) -> List[np.ndarray]:
        """Full tensor p = first d0*rest elements of concat_r slot_r[p's segment]
        (padding stripped).  bf16 -> uint16 bits, e4m3 -> uint8 codes."""
        lay = self.layouts[0]
        slot_bytes = 2 * lay.S if dtype == BF16 else lay.S_bytes_fp8
        fulls = []
        for m in lay.params:
            if dtype == FP8 and m.fp8_eligible:
                esize, boff, np_t = 1, m.byte_offset_fp8, np.uint8
            else:
                esize = 2
                boff = 2 * m.elem_offset if dtype == BF16 else m.byte_offset_fp8
                np_t = np.uint16
            pieces = [ag[r * slot_bytes + boff: r * slot_bytes + boff + m.padded_numel * esize]
                      for r in range(self.W)]
            flat = np.concatenate(pieces).view(np_t)[:m.numel]
            fulls.append(flat.reshape(m.shape).copy())
        return fulls

    def unshard(self, shards: Sequence[np.ndarray], dtype: str = BF16, scales=None):
        """copy-in on every rank -> all-gather -> copy-out.  Returns (ag_buffer, fulls);
        every rank holds the same ag_buffer and hence the same full tensors."""
        slots = [self.copy_in(s, dtype, scales) for s in shards]
        ag = self.all_gather(slots)
        return ag, self.copy_out(ag, dtype)

    # ------------------------------------------------------------ a7: RS copy-in
    def rs_copy_in(self, grads: Sequence[np.ndarray], grad_dtype: str = BF16,
                   mean: bool = True, reduce_dtype: str = FP32, divisor: int | None = None) -> np.ndarray:
        """One rank's reduce-scatter input [W][S]: row-chunk r of every full grad, widened to
        fp32 and divided once by W, zero padding elsewhere (reading R1).
        reduce_dtype bf16 (reading R11) rounds the pre-divided fp32 value to bf16.
        `divisor` (default W) is the number of ranks the mean runs over: the whole
        replicate x shard mesh under HSDP (reading R15)."""
        lay = self.layouts[0]
        buf = np.zeros(self.W * lay.S, dtype=np.float32)
        div = np.float32(self.W if divisor is None else divisor)
        for p, g in enumerate(grads):
            g32 = bf16_bits_to_f32(g).reshape(-1) if grad_dtype == BF16 else np.asarray(g, np.float32).reshape(-1)
            x = (g32 / div).astype(np.float32) if mean else g32
            for r in range(self.W):
                m = self.layouts[r].params[p]
                n = m.row_count * m.rest
                src = r * m.padded_numel
                dst = r * lay.S + m.elem_offset
                buf[dst:dst + n] = x[src:src + n]
        if reduce_dtype == BF16:
            return bf16_rne_bits(buf)
        return buf

    # --------------------------------------------------------- a8: reduce-scatter
    def reduce_scatter(self, inputs: Sequence[np.ndarray], reduce_dtype: str = FP32):
        """Per rank r: dict(order=fp32 ascending-rank sum,
        exact=correctly rounded fp32 of the exact sum, mag=sum_q |x_q| in fp64).
        For reduce_dtype bf16 the inputs are bf16 bits and `order` is the fp32 sum of the
        widened bf16 values (the hop-wise bf16 rounding of a real reducer is bounded in
        tests, reading R11)."""
        S = self.S
        outs = []
        for r in range(self.W):
            xs = []
            for q in range(self.W):
                chunk = inputs[q][r * S:(r + 1) * S]
                xs.append(bf16_bits_to_f32(chunk) if reduce_dtype == BF16 else np.asarray(chunk, np.float32))
            acc = xs[0].copy()
            for q in range(1, self.W):
                acc = (acc + xs[q]).astype(np.float32)
            X = np.stack([x.astype(np.float64) for x in xs])
            outs.append(dict(order=acc, exact=_exact_sum_to_f32(X), mag=np.abs(X).sum(axis=0)))
        return outs

    # --------------------------------------------------------- a9: RS copy-out
    def rs_copy_out(self, out: np.ndarray, rank: int) -> List[np.ndarray]:
        """Sharded grad p of `rank` = first rows*rest elements of out[off_p:], shape
        (rows, *shape[1:]) — empty for trailing empty shards."""
        res = []
        for m in self.layouts[rank].params:
            n = m.row_count * m.rest
            res.append(np.asarray(out[m.elem_offset:m.elem_offset + n]).reshape((m.row_count,) + m.shape[1:]).copy())
        return res

    def reduce_scatter_grads(self, grads_per_rank, grad_dtype: str = BF16, mean: bool = True,
                             reduce_dtype: str = FP32):
        """Full post-backward path: per rank a list of sharded grads for each reference
        ('order', 'exact') plus the magnitude sum 'mag' used by the tolerance (R10)."""
        inputs = [self.rs_copy_in(g, grad_dtype, mean, reduce_dtype) for g in grads_per_rank]
        outs = self.reduce_scatter(inputs, reduce_dtype)
        return [{k: self.rs_copy_out(o[k], r) for k in ("order", "exact", "mag")}
                for r, o in enumerate(outs)]


def _exact_sum_to_f32(X: np.ndarray) -> np.ndarray:
    """Correctly rounded fp32 of the exact column sums of fp32 values X[q, k].

    The fp64 sum is exact when the addends span < 2**26 in magnitude (24-bit significands
    plus carry bits fit in 53 bits for W <= 8); other columns use math.fsum (exact)."""
    s = X.sum(axis=0)
    absx = np.abs(X)
    nz = np.where(absx > 0, absx, np.inf).min(axis=0)
    mx = absx.max(axis=0)
    risky = np.nonzero((mx > 0) & (mx / nz >= 2.0 ** 26))[0]
    for k in risky:
        s[k] = math.fsum(X[:, k].tolist())
    return s.astype(np.float32)


def rs_error_ok(y: np.ndarray, exact: np.ndarray, mag: np.ndarray, W: int,
                rel: float = 1e-6):
    """Tolerance of reading R10: elementwise |y - exact| <= rel*mag + W*2**-149 and
    normwise ||y - exact|| / ||exact|| <= rel.  Returns (ok, worst_elem_ratio, norm_rel)."""
    y = np.asarray(y, np.float64)
    e = np.asarray(exact, np.float64)
    bound = rel * np.asarray(mag, np.float64) + W * 2.0 ** -149
    diff = np.abs(y - e)
    ratio = float(np.max(diff / bound)) if diff.size else 0.0
    nrm = float(np.linalg.norm(e))
    nrel = float(np.linalg.norm(y - e) / nrm) if nrm > 0 else float(np.linalg.norm(y - e))
    return (ratio <= 1.0 and nrel <= rel), ratio, nrel


class HsdpWorld:
    """HSDP (appendix:hsdp): a 2-D mesh of `replicate` replica groups x
    `shard` ranks; global rank g = replica * shard + shard_rank (replica dim outer, reading
    R15).  "each shard group runs FSDP and the replica group runs normal data parallel
    ... with the addition of backward gradient allreduce across replica groups"
    (PAPER.md:476): parameters are Shard(0) over the shard group, unshard is the shard
    group's all-gather, and the gradient is pre-divided by the whole world size
    ("HSDP adds all_reduce(mean via pre-division) across the replicate dim"),
    reduce-scattered inside each shard group, then all-reduced (sum) across replicas."""

    def __init__(self, shapes, replicate: int, shard: int, fp8_eligible=None):
        self.R, self.Ws = int(replicate), int(shard)
        self.W = self.R * self.Ws
        self.fsdp = World(shapes, self.Ws, fp8_eligible)   # one shard group (all replicas identical)

    def shard_rank(self, g: int) -> int:
        return g % self.Ws

    def replica(self, g: int) -> int:
        return g // self.Ws

    def reduce_scatter_grads(self, grads_per_rank, grad_dtype: str = BF16, mean: bool = True):
        """grads_per_rank[g] = global rank g's full grads.  Returns per global rank a dict of
        per-param sharded grads: 'order' (shard-group sum in ascending shard rank, then the
        replica sum in ascending replica), 'exact' (correctly rounded fp32 of the exact sum
        of all W pre-divided terms), 'mag' (sum of their magnitudes)."""
        w = self.fsdp
        inputs = [w.rs_copy_in(g, grad_dtype, mean, FP32, divisor=self.W) for g in grads_per_rank]
        # reduce-scatter inside every shard group
        per_rep = [w.reduce_scatter(inputs[r * self.Ws:(r + 1) * self.Ws]) for r in range(self.R)]
        S = w.S
        out = []
        for g in range(self.W):
            s = self.shard_rank(g)
            acc = per_rep[0][s]["order"].copy()
            for r in range(1, self.R):          # all-reduce across the replica group
                acc = (acc + per_rep[r][s]["order"]).astype(np.float32)
            X = np.stack([inputs[q][s * S:(s + 1) * S].astype(np.float64) for q in range(self.W)])
            res = dict(order=acc, exact=_exact_sum_to_f32(X), mag=np.abs(X).sum(axis=0))
            out.append({k: w.rs_copy_out(v, s) for k, v in res.items()})
        return out
