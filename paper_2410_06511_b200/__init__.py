"""B200-native FSDP2 per-parameter Shard(0) hot path (arXiv 2410.06511, TorchTitan).

The compute path is libfsdp_b200.so (hand-written sm_100a CUDA + NCCL behind the C ABI
in include/fsdp_b200.h); this package is its thin Python binding.  Importing it loads
the library and raises ImportError if it is not built — there is no CPU fallback.
"""
from ._capi import lib as _lib, FsdpError, LIB_PATH

_lib()  # fail loudly at import if the CUDA library is missing

from .fsdp import (Mesh, Layer, layout_compute, get_unique_id, fsdp_shard, precompute_fp8_scales,  # noqa: E402
                   fsdp_unshard, fsdp_wait_unshard, all_gather_params, fsdp_reshard,
                   reduce_scatter_grads, fsdp_wait_reduce_scatter, zero_grad, stage_copy_in,
                   stage_copy_out, stage_local_amax, stage_fp8_scale, stage_rs_copy_in,
                   stage_rs_copy_out, unsharded_layout, stage_unshard_push, grad_staging_layout,
                   stage_grads_to_staging, stage_rs_pull, stage_rs_pull_hsdp, stage_hsdp_piece_pull,
                   stage_hsdp_replica_gather, stage_rs_scatter,
                   stage_rs_recv_reduce)

__all__ = ["Mesh", "Layer", "layout_compute", "get_unique_id", "fsdp_shard", "precompute_fp8_scales",
           "fsdp_unshard", "fsdp_wait_unshard", "all_gather_params", "fsdp_reshard",
           "reduce_scatter_grads", "fsdp_wait_reduce_scatter", "zero_grad", "stage_copy_in",
           "stage_copy_out", "stage_local_amax", "stage_fp8_scale", "stage_rs_copy_in",
           "stage_rs_copy_out", "unsharded_layout", "stage_unshard_push", "grad_staging_layout",
           "stage_grads_to_staging", "stage_rs_pull", "stage_rs_pull_hsdp", "stage_hsdp_piece_pull",
           "stage_hsdp_replica_gather", "stage_rs_scatter",
           "stage_rs_recv_reduce", "FsdpError", "LIB_PATH"]
