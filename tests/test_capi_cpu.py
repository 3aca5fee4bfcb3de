"""C-ABI checks that need no GPU: the library loads, exports every symbol include/fsdp_b200.h
declares, and its host-side Shard(0) layout (component N1) equals the oracle's bit for bit."""
import ctypes
import os
import re

import numpy as np
import pytest

import synth
from oracle import unit_layout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fsdp_b200.h")


def _declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fsdp_[a-z0-9_]+)\s*\(", txt)))


def test_library_loads_and_exports_every_declared_symbol():
    import paper_2410_06511_b200 as f
    from paper_2410_06511_b200 import _capi
    lib = ctypes.CDLL(f.LIB_PATH)
    syms = _declared_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the binding declares every one of them with the same name
    bound = set(_capi.SIGNATURES) | set(_capi._OTHER)
    assert set(syms) == bound, set(syms) ^ bound
    assert _capi.lib().fsdp_abi_version() == 2


def test_library_is_sm100a():
    import subprocess
    import paper_2410_06511_b200 as f
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", f.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _check_against_oracle(shapes, elig, W):
    import paper_2410_06511_b200 as f
    hashes = set()
    for r in range(W):
        metas, S, Sb, h = f.layout_compute(shapes, W, r, elig)
        want = unit_layout(shapes, W, r, elig)
        assert S == want.S and Sb == want.S_bytes_fp8
        for m, w in zip(metas, want.params):
            assert m == {"dim0": w.dim0, "rest": w.rest, "chunk_rows": w.chunk_rows, "row_begin": w.row_begin,
                         "row_count": w.row_count, "padded_numel": w.padded_numel,
                         "elem_offset": w.elem_offset, "fp8_byte_offset": w.byte_offset_fp8}
        hashes.add(h)
    assert len(hashes) == 1   # every rank computes the same layout hash


def test_layout_bruteforce_vs_oracle():
    for W in range(1, 9):
        for d0 in range(0, 41, 3):
            for rest in (1, 3, 16):
                _check_against_oracle([(d0, rest), (5,), (d0 + 1, 2, 3)], [True, False, True], W)


@pytest.mark.parametrize("seed", range(6))
def test_layout_ragged_units_vs_oracle(seed):
    u = synth.ragged_unit(seed)
    for W in (1, 2, 3, 4, 5, 8):
        _check_against_oracle([s for _, s, _ in u], [e for _, _, e in u], W)


@pytest.mark.parametrize("name", ["toy", "llama3.1-8b", "llama3.1-70b"])
def test_layout_llama_vs_oracle(name):
    for u in synth.model_units(name)[-2:]:   # one block + root
        for W in (1, 2, 4, 8):
            _check_against_oracle([s for _, s, _ in u], [e for _, _, e in u], W)


def test_layout_hash_detects_mismatch():
    import paper_2410_06511_b200 as f
    h1 = f.layout_compute([(8, 4), (3,)], 2, 0)[3]
    h2 = f.layout_compute([(8, 5), (3,)], 2, 0)[3]
    h3 = f.layout_compute([(8, 4), (3,)], 2, 0, [True, False])[3]
    h4 = f.layout_compute([(8, 4), (3,)], 4, 0)[3]
    assert len({h1, h2, h3, h4}) == 4


def test_layout_errors():
    import paper_2410_06511_b200 as f
    with pytest.raises(f.FsdpError) as e:
        f.layout_compute([()], 2, 0)
    assert e.value.status_name == "FSDP_ERR_SHAPE"
    with pytest.raises(f.FsdpError) as e:
        f.layout_compute([(4,)], 2, 2)
    assert e.value.status_name == "FSDP_ERR_INVALID_ARGUMENT"
    with pytest.raises(f.FsdpError) as e:
        f.layout_compute([(4,)], 0, 0)
    assert e.value.status_name == "FSDP_ERR_INVALID_ARGUMENT"


def test_unique_id_without_gpu():
    import paper_2410_06511_b200 as f
    a, b = f.get_unique_id(), f.get_unique_id()
    assert len(a) == 128 and a != b


def _header_enums():
    """name -> value of every `NAME = <int>` enumerator in include/fsdp_b200.h."""
    txt = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    return {n: int(v) for n, v in re.findall(r"\b(FSDP_[A-Z0-9_]+)\s*=\s*(\d+)", txt)}


def test_binding_constants_match_header_enums():
    from paper_2410_06511_b200 import _capi as c
    e = _header_enums()
    for code, name in c.STATUS.items():
        assert e[name] == code, name
    assert (e["FSDP_FLOAT32"], e["FSDP_BFLOAT16"], e["FSDP_FLOAT8_E4M3FN"]) == (c.FLOAT32, c.BFLOAT16, c.FLOAT8_E4M3FN)
    assert (e["FSDP_ALGO_NCCL"], e["FSDP_ALGO_P2P"]) == (c.ALGO_NCCL, c.ALGO_P2P)
    assert (e["FSDP_P2P_RS_PULL"], e["FSDP_P2P_RS_STORE"], e["FSDP_P2P_RS_AUTO"]) == \
        (c.P2P_RS_PULL, c.P2P_RS_STORE, c.P2P_RS_AUTO)
    # profile kinds: the binding's names are in enum order and the struct arrays have NUM entries
    assert len(c.PROF_KINDS) == e["FSDP_PROF_NUM"]
    assert c.Profile.launches.size == 8 * e["FSDP_PROF_NUM"]
    assert e["FSDP_PROF_RS_SCATTER"] == c.PROF_KINDS.index("rs_scatter")
    assert e["FSDP_PROF_HANDSHAKE"] == c.PROF_KINDS.index("handshake")
