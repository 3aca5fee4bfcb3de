"""Float8 per-tensor scaling strategies — oracle (test infrastructure only).

PAPER.md:157: torchao.float8 "supports multiple per-tensor scaling strategies, including
dynamic, delayed, and static".  SPEC.md:417 defines them: "scale = E4M3_MAX / amax
(dynamic: current tensor amax; delayed: max of the amax history, history updated after
use; static: fixed)"; "Delayed-scaling history initialized with the first
observed amax; length default 16" (reading R16: the paper is silent on both).

* dynamic: ``World.precompute_fp8_scales`` (world.py).
* delayed: ``DelayedScaling`` below.
* static: a caller-given scale, passed straight to the cast (no oracle state).
"""
from __future__ import annotations

import numpy as np

from .casts import fp8_scale_from_amax


class DelayedScaling:
    """Per-parameter amax history of length H (ring buffer)."""

    def __init__(self, n_params: int, history_len: int = 16):
        self.H = int(history_len)
        self.hist = np.zeros((n_params, self.H), dtype=np.float32)
        self.init = np.zeros(n_params, dtype=bool)
        self.pos = np.zeros(n_params, dtype=np.int64)

    def step(self, amax_now: np.ndarray, eligible) -> np.ndarray:
        """One precompute: returns the scales to use now, then records amax_now."""
        amax_now = np.asarray(amax_now, dtype=np.float32)
        scale = np.zeros(len(amax_now), dtype=np.float32)
        for p, a in enumerate(amax_now):
            if not eligible[p]:
                continue
            if not self.init[p]:                     # initialised with the first amax
                self.hist[p, :] = a
                self.init[p] = True
            scale[p] = fp8_scale_from_amax(np.max(self.hist[p]))   # max of the history ...
            self.hist[p, self.pos[p]] = a                          # ... updated after use
            self.pos[p] = (self.pos[p] + 1) % self.H
        return scale
