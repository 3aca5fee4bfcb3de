"""ctypes declarations of include/fsdp_b200.h (argument marshalling only).

Loads the in-tree ``libfsdp_b200.so`` and fails loudly if it is missing: there is no
CPU or PyTorch fallback for any call."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfsdp_b200.so")

FSDP_MAX_NDIM = 8
FSDP_UNIQUE_ID_BYTES = 128

# fsdp_dtype_t
FLOAT32, BFLOAT16, FLOAT8_E4M3FN = 0, 1, 2

STATUS = {0: "FSDP_OK", 1: "FSDP_ERR_INVALID_ARGUMENT", 2: "FSDP_ERR_SHAPE", 3: "FSDP_ERR_DTYPE",
          4: "FSDP_ERR_STATE", 5: "FSDP_ERR_OUT_OF_MEMORY", 6: "FSDP_ERR_CUDA", 7: "FSDP_ERR_NCCL",
          8: "FSDP_ERR_TIMEOUT", 9: "FSDP_ERR_NONFINITE", 10: "FSDP_ERR_UNAVAILABLE"}

PROF_KINDS = ["copy_in", "all_gather", "copy_out", "rs_copy_in", "reduce_scatter", "rs_copy_out",
              "amax", "scale", "all_reduce", "unshard_push", "rs_pull", "stage_grads", "handshake",
              "rs_scatter", "rs_reduce", "replica_gather"]
ALGO_NCCL, ALGO_P2P = 0, 1
P2P_RS_PULL, P2P_RS_STORE, P2P_RS_AUTO = 0, 1, 2


class ParamDesc(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("fp8_eligible", C.c_int32), ("shape", C.c_int64 * FSDP_MAX_NDIM)]


class ParamMeta(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("dim0", "rest", "chunk_rows", "row_begin", "row_count",
                                         "padded_numel", "elem_offset", "fp8_byte_offset")]


class Profile(C.Structure):
    _fields_ = [("launches", C.c_int64 * 16), ("total_ms", C.c_double * 16), ("bytes", C.c_int64 * 16)]


class FsdpError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        self.status = status
        self.status_name = STATUS.get(status, str(status))
        super().__init__(f"{fn}: {self.status_name}: {msg}")


_VP = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_PP = C.POINTER(C.c_void_p)
# fsdp_alloc_fn / fsdp_free_fn (fsdp_mesh_set_allocator)
ALLOC_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_size_t, C.c_int32, C.POINTER(C.c_void_p))
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_int32)
HOSTAG_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

# name -> argtypes (restype is fsdp_status_t unless listed in _OTHER)
SIGNATURES = {
    "fsdp_layout_compute": [_I32, C.POINTER(ParamDesc), _I32, _I32, C.POINTER(ParamMeta), C.POINTER(_I64),
                            C.POINTER(_I64), C.POINTER(C.c_uint64)],
    "fsdp_get_unique_id": [C.POINTER(C.c_uint8)],
    "fsdp_mesh_init": [C.POINTER(C.c_uint8), _I32, _I32, _I32, C.POINTER(_VP)],
    "fsdp_mesh_init_local": [_I32, _I32, _I32, C.POINTER(_VP)],
    "fsdp_mesh_init_hsdp": [C.POINTER(C.c_uint8), _I32, _I32, _I32, _I32, C.POINTER(_VP)],
    "fsdp_mesh_info_hsdp": [_VP, C.POINTER(_I32), C.POINTER(_I32)],
    "fsdp_mesh_destroy": [_VP],
    "fsdp_mesh_info": [_VP, C.POINTER(_I32), C.POINTER(_I32), C.POINTER(_I32)],
    "fsdp_mesh_synchronize": [_VP, _I64],
    "fsdp_mesh_abort": [_VP],
    "fsdp_mesh_set_algo": [_VP, _I32],
    "fsdp_mesh_get_algo": [_VP, C.POINTER(_I32)],
    "fsdp_mesh_set_p2p_rs": [_VP, _I32],
    "fsdp_mesh_get_p2p_rs": [_VP, C.POINTER(_I32)],
    "fsdp_profile_enable": [_VP, _I32],
    "fsdp_profile_read": [_VP, C.POINTER(Profile), _I32],
    "fsdp_mesh_set_allocator": [_VP, ALLOC_FN, FREE_FN, _VP],
    "fsdp_shard": [_VP, _I32, C.POINTER(ParamDesc), _PP, C.POINTER(_VP)],
    "fsdp_layer_destroy": [_VP],
    "fsdp_layer_info": [_VP, C.POINTER(_I32), C.POINTER(_I64), C.POINTER(_I64)],
    "fsdp_param_meta": [_VP, _I32, C.POINTER(ParamMeta)],
    "fsdp_sharded_param": [_VP, _I32, C.POINTER(_VP)],
    "fsdp_sharded_flat": [_VP, C.POINTER(_VP)],
    "fsdp_precompute_fp8_scales": [_VP, _PP, _I32, _VP],
    "fsdp_precompute_fp8_scales_delayed": [_VP, _PP, _I32, _I32, _VP],
    "fsdp_fp8_scales": [_VP, C.POINTER(_VP), C.POINTER(_VP)],
    "fsdp_unshard": [_VP, _I32, _VP, _VP],
    "fsdp_wait_unshard": [_VP, _VP],
    "fsdp_all_gather_params": [_VP, _I32, _VP, _VP],
    "fsdp_unsharded_param": [_VP, _I32, C.POINTER(_VP), C.POINTER(_I32)],
    "fsdp_reshard": [_VP, _VP],
    "fsdp_reduce_scatter_grads": [_VP, _PP, _I32, _I32, _I32, _I32, _VP],
    "fsdp_wait_reduce_scatter": [_VP, _VP],
    "fsdp_full_grad_buffer": [_VP, _I32, _I32, C.POINTER(_VP)],
    "fsdp_sharded_grad": [_VP, _I32, C.POINTER(_VP)],
    "fsdp_sharded_grad_flat": [_VP, C.POINTER(_VP)],
    "fsdp_zero_grad": [_VP, _VP],
    "fsdp_stage_copy_in": [_VP, _I32, _VP, _VP, _VP, _VP],
    "fsdp_stage_copy_out": [_VP, _I32, _VP, _PP, _VP],
    "fsdp_stage_local_amax": [_VP, _VP, _VP],
    "fsdp_stage_fp8_scale": [_VP, _VP, _VP, _VP],
    "fsdp_stage_rs_copy_in": [_VP, _PP, _I32, _I32, _I32, _VP, _VP],
    "fsdp_stage_rs_copy_out": [_VP, _VP, _I32, _I32, _VP],
    "fsdp_unsharded_layout": [_VP, _I32, C.POINTER(_I64), C.POINTER(_I64)],
    "fsdp_stage_unshard_push": [_VP, _I32, _VP, _PP, _VP, _VP],
    "fsdp_grad_staging_layout": [_VP, C.POINTER(_I64), C.POINTER(_I64)],
    "fsdp_stage_grads_to_staging": [_VP, _PP, _I32, _VP, _VP],
    "fsdp_stage_rs_pull": [_VP, _PP, _I32, _I32, _I32, _I32, _VP],
    "fsdp_stage_rs_pull_hsdp": [_VP, _PP, _I32, _I32, _I32, _I32, _I32, _VP],
    "fsdp_mesh_get_hsdp_rs": [_VP, C.POINTER(_I32)],
    "fsdp_mesh_init_hostcoll": [_I32, _I32, _I32, _I32, HOSTAG_FN, _VP, C.POINTER(_VP)],
    "fsdp_stage_hsdp_piece_pull": [_VP, _PP, _I32, _I32, _I32, _I32, _I32, _VP, _VP],
    "fsdp_stage_hsdp_replica_gather": [_VP, _PP, _I32, _I32, _VP],
    "fsdp_mesh_memory": [_VP, C.POINTER(_I64)],
    "fsdp_stage_rs_scatter": [_VP, _PP, _I32, _PP, _I32, _VP],
    "fsdp_stage_rs_recv_reduce": [_VP, _VP, _PP, _I32, _I32, _I32, _I32, _VP],
}
_OTHER = {
    "fsdp_abi_version": ([], C.c_int32),
    "fsdp_last_error": ([], C.c_char_p),
    "fsdp_status_string": ([C.c_int], C.c_char_p),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: the CUDA library is not built (run __graft_entry__.build() or "
            f"python paper_2410_06511_b200/build.py). There is no CPU fallback.")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    for name, args in SIGNATURES.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    for name, (args, res) in _OTHER.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


def check(status: int, fn: str):
    if status != 0:
        msg = lib().fsdp_last_error()
        raise FsdpError(status, fn, msg.decode() if msg else "")


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)
