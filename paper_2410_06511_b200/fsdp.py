"""Thin Python binding of the C ABI (include/fsdp_b200.h): same names, torch tensors in,
pointers out.  Every step of the path runs in libfsdp_b200.so; this module only
marshals arguments, wraps library-owned device memory as torch views, and (in
``Mesh.from_process_group``) broadcasts the NCCL unique id over torch.distributed.

Names follow BASELINE.json / the paper's statement of the problem:
``fsdp_shard(params, mesh)``, ``fsdp_unshard`` / ``all_gather_params(layer, dtype,
fp8_scale)``, ``precompute_fp8_scales(params)``, ``reduce_scatter_grads(layer,
reduce_dtype, mean)``.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import torch

from . import _capi as capi
from ._capi import ParamDesc, ParamMeta, call

_DT = {torch.float32: capi.FLOAT32, torch.bfloat16: capi.BFLOAT16, torch.float8_e4m3fn: capi.FLOAT8_E4M3FN}
_DT_INV = {v: k for k, v in _DT.items()}


def _dtype_code(dt) -> int:
    if isinstance(dt, int):
        return dt
    if dt not in _DT:
        raise ValueError(f"unsupported dtype {dt}")
    return _DT[dt]


def _stream(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class _CAI:
    """__cuda_array_interface__ view of library-owned device memory (no copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None,
                                         "stream": None}


def _view(ptr: int, shape, dtype: torch.dtype, device: int) -> torch.Tensor:
    shape = tuple(int(s) for s in shape)
    n = 1
    for s in shape:
        n *= s
    if n == 0 or not ptr:
        return torch.empty(shape, dtype=dtype, device=f"cuda:{device}")
    if dtype == torch.float32:
        return torch.as_tensor(_CAI(ptr, shape, "<f4"), device=f"cuda:{device}")
    if dtype == torch.bfloat16:
        return torch.as_tensor(_CAI(ptr, shape, "<u2"), device=f"cuda:{device}").view(torch.bfloat16)
    if dtype == torch.float8_e4m3fn:
        return torch.as_tensor(_CAI(ptr, shape, "|u1"), device=f"cuda:{device}").view(torch.float8_e4m3fn)
    if dtype == torch.uint8:
        return torch.as_tensor(_CAI(ptr, shape, "|u1"), device=f"cuda:{device}")
    raise ValueError(dtype)


def _descs(shapes, fp8_eligible) -> C.Array:
    n = len(shapes)
    arr = (ParamDesc * max(n, 1))()
    for p, shape in enumerate(shapes):
        shape = tuple(int(s) for s in shape)
        arr[p].ndim = len(shape)
        arr[p].fp8_eligible = int(bool(fp8_eligible[p])) if fp8_eligible is not None else 0
        for i, s in enumerate(shape[:capi.FSDP_MAX_NDIM]):
            arr[p].shape[i] = s
    return arr


def _meta_dict(m: ParamMeta) -> dict:
    return {k: int(getattr(m, k)) for k, _ in ParamMeta._fields_}


# ----------------------------------------------------------------------- host-only
def layout_compute(shapes: Sequence[Sequence[int]], world_size: int, rank: int,
                   fp8_eligible: Optional[Sequence[bool]] = None):
    """Shard(0) metadata on the host (no GPU): (list of meta dicts, S, S_bytes_fp8, hash)."""
    n = len(shapes)
    descs = _descs(shapes, fp8_eligible)
    metas = (ParamMeta * max(n, 1))()
    S = C.c_int64()
    Sb = C.c_int64()
    h = C.c_uint64()
    call("fsdp_layout_compute", n, descs, world_size, rank, metas, C.byref(S), C.byref(Sb), C.byref(h))
    return [_meta_dict(metas[p]) for p in range(n)], S.value, Sb.value, h.value


def get_unique_id() -> bytes:
    buf = (C.c_uint8 * capi.FSDP_UNIQUE_ID_BYTES)()
    call("fsdp_get_unique_id", buf)
    return bytes(buf)


def _torch_allocator():
    """fsdp_alloc_fn / fsdp_free_fn backed by the torch caching allocator (SURVEY.md §8(b)
    "Ownership"): the library's bulk buffers show up in torch.cuda.memory_allocated() and
    share torch's cache.  The library synchronizes the device before every free."""
    def alloc(ctx, nbytes, dev, out):
        try:
            out[0] = torch.cuda.caching_allocator_alloc(int(nbytes), int(dev))
            return 0
        except Exception:          # OOM (or anything else): FSDP_ERR_OUT_OF_MEMORY in the caller
            return 1

    def free(ctx, ptr, dev):
        if ptr:
            torch.cuda.caching_allocator_delete(int(ptr))
    return capi.ALLOC_FN(alloc), capi.FREE_FN(free)


def _host_allgather(group):
    """fsdp_host_allgather_fn over a torch.distributed group (any backend; gloo keeps it on
    the CPU): the host-collective mesh's handle exchange, layout-hash check and barriers."""
    import torch.distributed as dist

    def fn(send, recv, nbytes, ctx):
        try:
            n = int(nbytes)
            W = dist.get_world_size(group)
            src = torch.frombuffer(bytearray(C.string_at(send, n)), dtype=torch.uint8) if n else \
                torch.empty(0, dtype=torch.uint8)
            out = [torch.empty(n, dtype=torch.uint8) for _ in range(W)]
            dist.all_gather(out, src, group=group)
            C.memmove(recv, torch.cat(out).numpy().tobytes(), n * W)
            return 0
        except Exception:   # noqa: BLE001 — reported as FSDP_ERR_UNAVAILABLE by the library
            return 1
    return capi.HOSTAG_FN(fn)


# ----------------------------------------------------------------------- mesh
class Mesh:
    """1-D data-parallel mesh (fsdp_mesh_t).  world_size defaults to all ranks."""

    def __init__(self, world_size: int, rank: int, device: int, unique_id: Optional[bytes] = None,
                 local: bool = False, shard_size: Optional[int] = None, allocator: str = "torch",
                 host_group=None):
        """world_size ranks; shard_size < world_size makes an HSDP mesh of world_size //
        shard_size replica groups x shard_size ranks.  allocator:
        "torch" (bulk buffers from the torch caching allocator, fsdp_mesh_set_allocator) or
        "cuda" (the library's own cudaMalloc).  host_group: a torch.distributed group (e.g.
        gloo) -> a host-collective P2P mesh with no NCCL (fsdp_mesh_init_hostcoll); its ranks
        may share a GPU."""
        if allocator not in ("torch", "cuda"):
            raise ValueError("allocator must be 'torch' or 'cuda'")
        self.world_size, self.rank, self.device = int(world_size), int(rank), int(device)
        self.local = local
        h = C.c_void_p()
        self._hostag = None
        self.hostcoll = host_group is not None
        if host_group is not None:
            self._hostag = _host_allgather(host_group)   # kept alive until destroy
            call("fsdp_mesh_init_hostcoll", self.world_size, self.rank, int(shard_size or 0), self.device,
                 self._hostag, None, C.byref(h))
        elif local:
            call("fsdp_mesh_init_local", self.world_size, self.rank, self.device, C.byref(h))
        else:
            if unique_id is None or len(unique_id) != capi.FSDP_UNIQUE_ID_BYTES:
                raise ValueError("unique_id of 128 bytes required")
            idb = (C.c_uint8 * capi.FSDP_UNIQUE_ID_BYTES).from_buffer_copy(unique_id)
            if shard_size is not None and shard_size != world_size:
                call("fsdp_mesh_init_hsdp", idb, self.world_size, self.rank, int(shard_size), self.device, C.byref(h))
            else:
                call("fsdp_mesh_init", idb, self.world_size, self.rank, self.device, C.byref(h))
        self.handle = h
        self.layers: List["Layer"] = []
        self.allocator = allocator
        self._alloc_cbs = None           # kept alive for the mesh's lifetime (frees at destroy)
        if allocator == "torch":
            self._alloc_cbs = _torch_allocator()
            call("fsdp_mesh_set_allocator", h, self._alloc_cbs[0], self._alloc_cbs[1], None)
        R = C.c_int32()
        rep = C.c_int32()
        call("fsdp_mesh_info_hsdp", h, C.byref(R), C.byref(rep))
        self.replicate_size, self.replica = R.value, rep.value
        self.shard_size = self.world_size // self.replicate_size
        self.shard_rank = self.rank % self.shard_size

    @classmethod
    def from_process_group(cls, group=None, device: Optional[int] = None,
                           shard_size: Optional[int] = None, allocator: str = "torch") -> "Mesh":
        """Collective: rank 0 creates the NCCL unique id, torch.distributed broadcasts it
        (the binding's only torch.distributed use), every rank initialises the mesh.
        shard_size (data_parallel_shard_degree) defaults to all ranks."""
        import torch.distributed as dist
        if device is None:
            device = torch.cuda.current_device()
        W = dist.get_world_size(group)
        r = dist.get_rank(group)
        obj = [get_unique_id() if r == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return cls(W, r, device, unique_id=obj[0], shard_size=shard_size, allocator=allocator)

    @property
    def algo(self) -> str:
        a = C.c_int32()
        call("fsdp_mesh_get_algo", self.handle, C.byref(a))
        return "p2p" if a.value == capi.ALGO_P2P else "nccl"

    def set_algo(self, algo: str):
        """Collective: 'nccl' (copy-in -> NCCL -> copy-out) or 'p2p' (fused NVLink kernels)."""
        call("fsdp_mesh_set_algo", self.handle, capi.ALGO_P2P if algo == "p2p" else capi.ALGO_NCCL)

    @property
    def hsdp_rs(self) -> str:
        """HSDP reduce-scatter mechanism on one NVSwitch domain: 'world_pull_2phase' (each
        replica reduces 1/R of the shard over all ranks, then the replicas exchange the
        finished pieces; default), 'world_pull' (one pull of the whole shard over all ranks),
        both nested-order sums; or 'rs+allreduce' (shard-group RS, then NCCL all-reduce)."""
        a = C.c_int32()
        call("fsdp_mesh_get_hsdp_rs", self.handle, C.byref(a))
        return {2: "world_pull_2phase", 1: "world_pull"}.get(a.value, "rs+allreduce")

    @property
    def p2p_rs(self) -> str:
        a = C.c_int32()
        call("fsdp_mesh_get_p2p_rs", self.handle, C.byref(a))
        return {capi.P2P_RS_STORE: "store", capi.P2P_RS_PULL: "pull"}.get(a.value, "auto")

    def set_p2p_rs(self, mode: str):
        """Collective: how the P2P reduce-scatter moves data — 'store' (peers store rows into
        each owner's receive buffer, local reduce), 'pull' (owners load rows from peers) or
        'auto' (pull at W = 2 for layers with zero-copy grad buffers, else store)."""
        codes = {"store": capi.P2P_RS_STORE, "pull": capi.P2P_RS_PULL, "auto": capi.P2P_RS_AUTO}
        if mode not in codes:
            raise ValueError("mode must be 'store', 'pull' or 'auto'")
        call("fsdp_mesh_set_p2p_rs", self.handle, codes[mode])

    def synchronize(self, timeout_ms: int = 0):
        call("fsdp_mesh_synchronize", self.handle, int(timeout_ms))

    def abort(self):
        """Rank-local: abort the communicators; layers/mesh can then be destroyed without
        any collective step (after FSDP_ERR_TIMEOUT / FSDP_ERR_NCCL on any rank)."""
        call("fsdp_mesh_abort", self.handle)

    def profile_enable(self, on: bool = True):
        call("fsdp_profile_enable", self.handle, int(bool(on)))

    def profile_read(self, reset: bool = True) -> dict:
        pr = capi.Profile()
        call("fsdp_profile_read", self.handle, C.byref(pr), int(bool(reset)))
        return {k: {"launches": int(pr.launches[i]), "ms": float(pr.total_ms[i]), "bytes": int(pr.bytes[i])}
                for i, k in enumerate(capi.PROF_KINDS)}

    def memory(self) -> dict:
        """Device bytes the mesh holds (fsdp_mesh_memory)."""
        out = (C.c_int64 * 4)()
        call("fsdp_mesh_memory", self.handle, out)
        return {"symmetric": out[0], "peer_mapped": out[1], "pools": out[2], "layers": out[3]}

    def destroy(self):
        for l in list(self.layers):
            l.destroy()
        if self.handle:
            call("fsdp_mesh_destroy", self.handle)
            self.handle = None


# ----------------------------------------------------------------------- layer
class Layer:
    """One FSDP unit (fsdp_layer_t).  Tensor accessors return views of library memory."""

    def __init__(self, mesh: Mesh, handle: C.c_void_p, shapes, fp8_eligible):
        self.mesh = mesh
        self.handle = handle
        self.shapes = [tuple(int(s) for s in sh) for sh in shapes]
        self.fp8_eligible = [bool(e) for e in fp8_eligible]
        n = C.c_int32()
        S = C.c_int64()
        Sb = C.c_int64()
        call("fsdp_layer_info", handle, C.byref(n), C.byref(S), C.byref(Sb))
        self.P, self.S, self.S_bytes_fp8 = n.value, S.value, Sb.value
        self.metas = [self.meta(p) for p in range(self.P)]
        self._pending_grads = None
        self._unshard_dtype = None

    @property
    def device(self) -> int:
        return self.mesh.device

    def meta(self, p: int) -> dict:
        m = ParamMeta()
        call("fsdp_param_meta", self.handle, p, C.byref(m))
        return _meta_dict(m)

    def sharded_flat(self) -> torch.Tensor:
        ptr = C.c_void_p()
        call("fsdp_sharded_flat", self.handle, C.byref(ptr))
        return _view(ptr.value, (self.S,), torch.float32, self.device)

    def sharded_param(self, p: int, padded: bool = False) -> torch.Tensor:
        """fp32 local shard of param p: (row_count, *shape[1:]) (or the padded chunk)."""
        ptr = C.c_void_p()
        call("fsdp_sharded_param", self.handle, p, C.byref(ptr))
        m = self.metas[p]
        rows = m["chunk_rows"] if padded else m["row_count"]
        return _view(ptr.value, (rows,) + self.shapes[p][1:], torch.float32, self.device)

    def sharded_grad_flat(self) -> torch.Tensor:
        ptr = C.c_void_p()
        call("fsdp_sharded_grad_flat", self.handle, C.byref(ptr))
        return _view(ptr.value, (self.S,), torch.float32, self.device)

    def sharded_grad(self, p: int) -> torch.Tensor:
        ptr = C.c_void_p()
        call("fsdp_sharded_grad", self.handle, p, C.byref(ptr))
        m = self.metas[p]
        return _view(ptr.value, (m["row_count"],) + self.shapes[p][1:], torch.float32, self.device)

    def unsharded_param(self, p: int) -> torch.Tensor:
        ptr = C.c_void_p()
        dt = C.c_int32()
        call("fsdp_unsharded_param", self.handle, p, C.byref(ptr), C.byref(dt))
        return _view(ptr.value, self.shapes[p], _DT_INV[dt.value], self.device)

    def unsharded_params(self) -> List[torch.Tensor]:
        return [self.unsharded_param(p) for p in range(self.P)]

    def full_grad_buffers(self, dtype=torch.bfloat16) -> List[torch.Tensor]:
        """Zero-copy gradients: views of the layer's own (symmetric, under P2P) full-grad
        buffer, one tensor per param with its full shape.  Writing the backward's grads
        here lets reduce_scatter_grads skip its staging copy (collective on first call)."""
        out = []
        for p in range(self.P):
            ptr = C.c_void_p()
            call("fsdp_full_grad_buffer", self.handle, _dtype_code(dtype), p, C.byref(ptr))
            out.append(_view(ptr.value, self.shapes[p], dtype, self.device))
        return out

    def sharded_state_dict(self, names: Optional[Sequence[str]] = None) -> dict:
        """Per-param local shards with their Shard(0) placement, without any communication
        ("allowing sharded state dict to be represented by DTensor without any
        communication"): {name: {"local": fp32 view (row_count, *shape[1:]), "global_shape",
        "row_begin", "world_size", "rank"}}.  The views alias the optimizer-visible shard."""
        names = names or [f"p{p}" for p in range(self.P)]
        out = {}
        for p, name in enumerate(names):
            m = self.metas[p]
            out[name] = {"local": self.sharded_param(p), "global_shape": self.shapes[p],
                         "row_begin": m["row_begin"], "world_size": self.mesh.shard_size
                         if hasattr(self.mesh, "shard_size") else self.mesh.world_size,
                         "rank": getattr(self.mesh, "shard_rank", self.mesh.rank)}
        return out

    def load_sharded_state_dict(self, state: dict, names: Optional[Sequence[str]] = None):
        """Copies local shards produced by sharded_state_dict (same world size and layout)
        back into the layer's fp32 shard; rows are checked against this rank's placement."""
        names = names or [f"p{p}" for p in range(self.P)]
        for p, name in enumerate(names):
            ent = state[name]
            m = self.metas[p]
            if tuple(ent["global_shape"]) != self.shapes[p] or int(ent["row_begin"]) != m["row_begin"]:
                raise ValueError(f"{name}: placement does not match this rank's Shard(0) layout")
            self.sharded_param(p).copy_(torch.as_tensor(ent["local"]).to(self.sharded_param(p).device))

    def fp8_scales(self):
        s = C.c_void_p()
        a = C.c_void_p()
        call("fsdp_fp8_scales", self.handle, C.byref(s), C.byref(a))
        return _view(s.value, (self.P,), torch.float32, self.device), _view(a.value, (self.P,), torch.float32, self.device)

    def destroy(self):
        if self.handle:
            call("fsdp_layer_destroy", self.handle)
            self.handle = None
            if self in self.mesh.layers:
                self.mesh.layers.remove(self)


def _ptr_array(tensors) -> C.Array:
    arr = (C.c_void_p * max(len(tensors), 1))()
    for i, t in enumerate(tensors):
        if t is None:
            arr[i] = None
        elif isinstance(t, torch.Tensor):
            if not t.is_contiguous():
                raise ValueError("tensors must be contiguous")
            arr[i] = t.data_ptr() if t.numel() else None
        else:  # numpy array (host)
            arr[i] = t.ctypes.data if t.size else None
    return arr


# ----------------------------------------------------------------------- API
def fsdp_shard(mesh: Mesh, params, fp8_eligible: Optional[Sequence[bool]] = None, shapes=None) -> Layer:
    """fsdp_shard(params, mesh): params = full fp32 tensors (host or device, contiguous) or
    None (then `shapes` gives the shapes and the shard starts at zero)."""
    if params is None:
        if shapes is None:
            raise ValueError("give params or shapes")
        full = None
    else:
        shapes = [tuple(p.shape) for p in params]
        for p in params:
            if isinstance(p, torch.Tensor) and p.dtype != torch.float32:
                raise ValueError("full params must be fp32 (the master copy)")
        full = _ptr_array(params)
    if fp8_eligible is None:
        fp8_eligible = [False] * len(shapes)
    descs = _descs(shapes, fp8_eligible)
    h = C.c_void_p()
    call("fsdp_shard", mesh.handle, len(shapes), descs, full, C.byref(h))
    layer = Layer(mesh, h, shapes, fp8_eligible)
    mesh.layers.append(layer)
    return layer


def precompute_fp8_scales(mesh: Mesh, layers: Sequence[Layer], stream=None, history_len: int = 0):
    """Per-tensor fp8 scales of every eligible param of `layers`: dynamic
    scaling by default, delayed scaling over an amax history when history_len > 0."""
    arr = (C.c_void_p * max(len(layers), 1))(*[l.handle.value for l in layers])
    if history_len > 0:
        call("fsdp_precompute_fp8_scales_delayed", mesh.handle, arr, len(layers), int(history_len), _stream(stream))
    else:
        call("fsdp_precompute_fp8_scales", mesh.handle, arr, len(layers), _stream(stream))


def fsdp_unshard(layer: Layer, dtype=torch.bfloat16, fp8_scales: Optional[torch.Tensor] = None, stream=None):
    sp = C.c_void_p(fp8_scales.data_ptr()) if fp8_scales is not None else C.c_void_p()
    call("fsdp_unshard", layer.handle, _dtype_code(dtype), sp, _stream(stream))
    layer._unshard_dtype = dtype


def fsdp_wait_unshard(layer: Layer, stream=None):
    call("fsdp_wait_unshard", layer.handle, _stream(stream))


def all_gather_params(layer: Layer, dtype=torch.bfloat16, fp8_scales: Optional[torch.Tensor] = None,
                      stream=None) -> List[torch.Tensor]:
    """fsdp_unshard + fsdp_wait_unshard; returns the per-param full tensors (views)."""
    sp = C.c_void_p(fp8_scales.data_ptr()) if fp8_scales is not None else C.c_void_p()
    call("fsdp_all_gather_params", layer.handle, _dtype_code(dtype), sp, _stream(stream))
    return layer.unsharded_params()


def fsdp_reshard(layer: Layer, stream=None):
    call("fsdp_reshard", layer.handle, _stream(stream))


def reduce_scatter_grads(layer: Layer, grads: Sequence[torch.Tensor], reduce_dtype=torch.float32,
                         mean: bool = True, accumulate: bool = False, stream=None):
    """Post-backward: this rank's full grads -> its fp32 sharded grads (pre-divided by W
    when mean).  The grads are kept referenced until fsdp_wait_reduce_scatter."""
    gd = grads[0].dtype
    if any(g.dtype != gd for g in grads):
        raise ValueError("all grads of a unit must share a dtype")
    arr = _ptr_array(grads)
    call("fsdp_reduce_scatter_grads", layer.handle, arr, _dtype_code(gd), _dtype_code(reduce_dtype),
         int(bool(mean)), int(bool(accumulate)), _stream(stream))
    layer._pending_grads = list(grads)


def fsdp_wait_reduce_scatter(layer: Layer, stream=None):
    call("fsdp_wait_reduce_scatter", layer.handle, _stream(stream))
    layer._pending_grads = None


def zero_grad(layer: Layer, stream=None):
    call("fsdp_zero_grad", layer.handle, _stream(stream))


# ----------------------------------------------------------------------- stage entry points
def stage_copy_in(layer: Layer, dtype, slot: torch.Tensor, fp8_scales: Optional[torch.Tensor] = None, stream=None,
                  amax_accum: Optional[torch.Tensor] = None):
    """amax_accum (float32 [P], fp8 only): max-accumulates the cast elements' |x| per param."""
    sp = C.c_void_p(fp8_scales.data_ptr()) if fp8_scales is not None else C.c_void_p()
    ap = C.c_void_p(amax_accum.data_ptr()) if amax_accum is not None else C.c_void_p()
    call("fsdp_stage_copy_in", layer.handle, _dtype_code(dtype), sp, C.c_void_p(slot.data_ptr()), ap,
         _stream(stream))


def stage_copy_out(layer: Layer, dtype, ag: torch.Tensor, outs: Sequence[torch.Tensor], stream=None):
    call("fsdp_stage_copy_out", layer.handle, _dtype_code(dtype), C.c_void_p(ag.data_ptr()), _ptr_array(outs),
         _stream(stream))


def stage_local_amax(layer: Layer, amax_out: torch.Tensor, stream=None):
    call("fsdp_stage_local_amax", layer.handle, C.c_void_p(amax_out.data_ptr()), _stream(stream))


def stage_fp8_scale(layer: Layer, amax: torch.Tensor, scale_out: torch.Tensor, stream=None):
    call("fsdp_stage_fp8_scale", layer.handle, C.c_void_p(amax.data_ptr()), C.c_void_p(scale_out.data_ptr()),
         _stream(stream))


def stage_rs_copy_in(layer: Layer, grads, reduce_dtype, mean: bool, rs_in: torch.Tensor, stream=None):
    call("fsdp_stage_rs_copy_in", layer.handle, _ptr_array(grads), _dtype_code(grads[0].dtype),
         _dtype_code(reduce_dtype), int(bool(mean)), C.c_void_p(rs_in.data_ptr()), _stream(stream))


def stage_rs_copy_out(layer: Layer, rs_out: torch.Tensor, reduce_dtype, accumulate: bool, stream=None):
    call("fsdp_stage_rs_copy_out", layer.handle, C.c_void_p(rs_out.data_ptr()), _dtype_code(reduce_dtype),
         int(bool(accumulate)), _stream(stream))


# ----------------------------------------------------------------------- P2P stage entry points
def unsharded_layout(layer: Layer, dtype=torch.bfloat16):
    """(byte offset of every param in the unsharded arena, arena bytes)."""
    offs = (C.c_int64 * max(layer.P, 1))()
    tot = C.c_int64()
    call("fsdp_unsharded_layout", layer.handle, _dtype_code(dtype), offs, C.byref(tot))
    return [int(offs[p]) for p in range(layer.P)], tot.value


def stage_unshard_push(layer: Layer, dtype, arenas: Sequence[torch.Tensor], fp8_scales: Optional[torch.Tensor] = None,
                       stream=None, amax_accum: Optional[torch.Tensor] = None):
    """amax_accum (float32 [P], fp8 only): max-accumulates the cast elements' |x| per param."""
    sp = C.c_void_p(fp8_scales.data_ptr()) if fp8_scales is not None else C.c_void_p()
    ap = C.c_void_p(amax_accum.data_ptr()) if amax_accum is not None else C.c_void_p()
    call("fsdp_stage_unshard_push", layer.handle, _dtype_code(dtype), sp, _ptr_array(arenas), ap, _stream(stream))


def grad_staging_layout(layer: Layer):
    offs = (C.c_int64 * max(layer.P, 1))()
    tot = C.c_int64()
    call("fsdp_grad_staging_layout", layer.handle, offs, C.byref(tot))
    return [int(offs[p]) for p in range(layer.P)], tot.value


def stage_grads_to_staging(layer: Layer, grads: Sequence[torch.Tensor], staging: torch.Tensor, stream=None):
    call("fsdp_stage_grads_to_staging", layer.handle, _ptr_array(grads), _dtype_code(grads[0].dtype),
         C.c_void_p(staging.data_ptr()), _stream(stream))


def stage_rs_pull(layer: Layer, stagings: Sequence[torch.Tensor], grad_dtype, reduce_dtype=torch.float32,
                  mean: bool = True, accumulate: bool = False, stream=None):
    call("fsdp_stage_rs_pull", layer.handle, _ptr_array(stagings), _dtype_code(grad_dtype),
         _dtype_code(reduce_dtype), int(bool(mean)), int(bool(accumulate)), _stream(stream))


def stage_rs_pull_hsdp(layer: Layer, stagings: Sequence[torch.Tensor], replicate: int, grad_dtype,
                       reduce_dtype=torch.float32, mean: bool = True, accumulate: bool = False, stream=None):
    """HSDP world pull: stagings[g] = global rank g's staging (g = replica * W + shard rank);
    grad (+)= sum over replicas of (sum over shard ranks of fp32(x) / (replicate * W))."""
    call("fsdp_stage_rs_pull_hsdp", layer.handle, _ptr_array(stagings), int(replicate), _dtype_code(grad_dtype),
         _dtype_code(reduce_dtype), int(bool(mean)), int(bool(accumulate)), _stream(stream))


def stage_hsdp_piece_pull(layer: Layer, stagings: Sequence[torch.Tensor], replicate: int, replica: int, grad_dtype,
                          res: torch.Tensor, reduce_dtype=torch.float32, mean: bool = True, stream=None):
    """HSDP two-phase RS, phase 1: res (fp32 [S]) = the nested world sum over piece `replica`."""
    call("fsdp_stage_hsdp_piece_pull", layer.handle, _ptr_array(stagings), int(replicate), int(replica),
         _dtype_code(grad_dtype), _dtype_code(reduce_dtype), int(bool(mean)), C.c_void_p(res.data_ptr()),
         _stream(stream))


def stage_hsdp_replica_gather(layer: Layer, res: Sequence[torch.Tensor], accumulate: bool = False, stream=None):
    """HSDP two-phase RS, phase 2: grad (+)= piece q from res[q] (replica q's phase-1 buffer)."""
    call("fsdp_stage_hsdp_replica_gather", layer.handle, _ptr_array(res), len(res), int(bool(accumulate)),
         _stream(stream))


def stage_rs_scatter(layer: Layer, grads: Sequence[torch.Tensor], recvs: Sequence[torch.Tensor],
                     include_self: bool = True, stream=None):
    """Store RS sender: this rank's rows of every rank r's chunk -> recvs[r] at slot `rank`
    (each receive buffer: W * S elements of the grads' dtype); include_self=False skips the
    own chunk (the receiver reads it from its grads)."""
    call("fsdp_stage_rs_scatter", layer.handle, _ptr_array(grads), _dtype_code(grads[0].dtype),
         _ptr_array(recvs), int(bool(include_self)), _stream(stream))


def stage_rs_recv_reduce(layer: Layer, recv: torch.Tensor, grad_dtype, reduce_dtype=torch.float32,
                         mean: bool = True, accumulate: bool = False, own_grads: Optional[Sequence[torch.Tensor]] = None,
                         stream=None):
    """Store RS receiver: grad (+)= ascending-rank fp32 sum over the W slots of recv / W; with
    own_grads, this rank's own rows come from its full grads instead of slot `rank`."""
    own = _ptr_array(own_grads) if own_grads is not None else None
    call("fsdp_stage_rs_recv_reduce", layer.handle, C.c_void_p(recv.data_ptr()), own, _dtype_code(grad_dtype),
         _dtype_code(reduce_dtype), int(bool(mean)), int(bool(accumulate)), _stream(stream))
