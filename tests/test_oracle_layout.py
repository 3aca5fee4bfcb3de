"""Pins for oracle/layout.py and World.shard — CPU only.

Pinned against: SPEC worked examples (tests/golden/spec_examples.json), hand-computed
Llama closed forms (tests/golden/layout_closed_forms.json), torch.chunk's row split
(library routine), brute force over small shapes, and the concat invariant
("concatenating the shards reproduces the original parameters", BASELINE.json)."""
import json
import os

import numpy as np
import pytest
import torch

import synth
from oracle import World, unit_layout
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SPEC = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))
CLOSED = json.load(open(os.path.join(GOLDEN, "layout_closed_forms.json")))


def test_spec_shard_2x2():
    ex = SPEC["shard0_2x2"]
    full = np.array(ex["full"], dtype=np.float32)
    w = World([full.shape], ex["world_size"])
    shards = w.shard([full])
    for r, want in enumerate(ex["rank_rows"]):
        m = w.layouts[r].params[0]
        got = shards[r][m.elem_offset:m.elem_offset + m.row_count * m.rest].reshape(m.row_count, m.rest)
        np.testing.assert_array_equal(got, np.array(want, dtype=np.float32))


def test_spec_uneven_rows():
    ex = SPEC["shard0_uneven"]
    counts = [unit_layout([(ex["dim0"],)], ex["world_size"], r).params[0].row_count
              for r in range(ex["world_size"])]
    assert counts == ex["row_counts"]


@pytest.mark.parametrize("W", [1, 2, 3, 4, 5, 6, 7, 8])
def test_row_split_matches_torch_chunk(W):
    for d0 in range(0, 41):
        t = torch.arange(d0)
        chunks = [len(c) for c in torch.chunk(t, W, dim=0)] if d0 > 0 else []
        chunks = chunks + [0] * (W - len(chunks))
        ours = [unit_layout([(d0, 3)], W, r).params[0].row_count for r in range(W)]
        assert ours == chunks, (d0, W)


def test_bruteforce_metadata_and_concat_invariant():
    rng = np.random.default_rng(0)
    for W in range(1, 9):
        for d0 in range(0, 41):
            for rest in (1, 3, 16):
                full = rng.standard_normal((d0, rest)).astype(np.float32)
                w = World([(d0, rest), (3,)], W)
                shards = w.shard([full, np.ones(3, np.float32)])
                rows = []
                begin = 0
                for r in range(W):
                    m = w.layouts[r].params[0]
                    assert m.row_begin == begin            # contiguous, ascending ranks
                    assert 0 <= m.row_count <= m.chunk_rows
                    assert m.padded_numel == m.chunk_rows * rest
                    assert m.elem_offset % 16 == 0
                    seg = shards[r][m.elem_offset:m.elem_offset + m.padded_numel]
                    rows.append(seg[:m.row_count * rest])
                    pad = seg[m.row_count * rest:]
                    assert np.all(pad.view(np.uint32) == 0)  # +0.0 bit pattern (c2)
                    begin += m.row_count
                    # second param starts after the aligned first segment
                    assert w.layouts[r].params[1].elem_offset == -(-m.padded_numel // 16) * 16
                assert begin == d0
                np.testing.assert_array_equal(np.concatenate(rows).reshape(d0, rest), full)


def _block_S(name, W):
    unit = synth.model_units(name, include_root=False)[0]
    shapes = [s for _, s, _ in unit]
    elig = [e for _, _, e in unit]
    return unit_layout(shapes, W, 0, elig)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_llama8b_closed_form(W):
    lay = _block_S("llama3.1-8b", W)
    assert lay.S == CLOSED["llama3.1-8b_block"][str(W)]
    if W == 8:
        assert [m.padded_numel for m in lay.params] == CLOSED["llama3.1-8b_block_shard_numels_w8"]
        assert lay.S_bytes_fp8 == CLOSED["llama3.1-8b_block_fp8_bytes_w8"]


def test_llama70b_and_toy_closed_form():
    assert _block_S("llama3.1-70b", 8).S == CLOSED["llama3.1-70b_block"]["8"]
    assert _block_S("toy", 2).S == CLOSED["toy_block"]["2"]
    for name, key in (("toy", "toy_total_params"), ("llama3.1-8b", "llama3.1-8b_total_params"),
                      ("llama3.1-70b", "llama3.1-70b_total_params")):
        total = sum(int(np.prod(s)) for u in synth.model_units(name) for _, s, _ in u)
        assert total == CLOSED[key]


def test_zero_dim_rejected():
    with pytest.raises(ValueError):
        unit_layout([()], 2, 0)
