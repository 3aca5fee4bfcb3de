/*
 * fsdp_b200.h — C ABI of the B200-native FSDP2 per-parameter Shard(0) hot path.
 *
 * The paper (arXiv 2410.06511, /root/reference/PAPER.md, cited "P:<line>") states the
 * problem as
 *   fully_shard(block, mesh=dp_mesh, mp_policy=MixedPrecisionPolicy(param_dtype,
 *               reduce_dtype), reshard_after_forward=...)
 * with parameters "represented as DTensors sharded on the tensor dimension 0"
 * (P:460), a bf16 parameter all-gather and an fp32 gradient reduce-scatter (P:154,
 * P:417), "only a single division kernel ... pre-dividing the local FP32
 * reduce-scatter gradient by world size", multi-tensor all-gather /
 * reduce-scatter kernels, "Float8 all-gather" with per-tensor scaling
 * (P:157), deterministic memory release without record_stream and the data-
 * parallel degree defaulting to all GPUs.  The calls below follow that
 * statement: fsdp_shard(params, mesh), fsdp_unshard / fsdp_all_gather_params(layer,
 * dtype, fp8_scale), fsdp_precompute_fp8_scales(params), fsdp_reduce_scatter_grads(
 * layer, reduce_dtype, mean).
 *
 * Conventions (all functions):
 *  - Every function returns fsdp_status_t; no C++ exception crosses the ABI.  On a
 *    non-OK status fsdp_last_error() returns a thread-local message.  Argument, shape,
 *    dtype and state errors are detected before any side effect.
 *  - Pointers named *_dev are CUDA device pointers (or, where stated, any pointer
 *    cudaMemcpyDefault accepts).  Streams are cudaStream_t passed as void*; NULL is the
 *    legacy default stream.
 *  - "Stream-ordered" calls return immediately; their device work is ordered after all
 *    work previously enqueued on `compute`, and later work on `compute` may consume
 *    the results after the matching fsdp_wait_* call.
 *  - A mesh and its layers are used from one host thread.
 *  - CUDA graphs: every stream-ordered call (precompute, unshard / wait / reshard,
 *    reduce-scatter / wait) may be captured while `compute` is capturing (e.g.
 *    torch.cuda.graph) and the graph replayed on the same stream, provided the same call
 *    sequence ran eagerly once before the capture (the capture uses the buffers that run
 *    allocated; pools never grow inside a capture -> FSDP_ERR_STATE) and the capture
 *    starts after a device synchronize.  P2P handshakes advance device-side epoch
 *    counters, so every replay re-synchronizes the ranks; every rank must replay the same
 *    graphs in the same order as its peers, like any collective.  Profiling events are not
 *    recorded inside a capture.
 *  - Layout: param order is the caller's order; rank r owns rows
 *    [min(r*c, d0), min((r+1)*c, d0)) with c = ceil(d0/W) (trailing ranks may be
 *    empty); the padded shard of param p has n_p = c*rest elements (rest = product of
 *    the non-leading dims) and sits at elem_offset off_p = sum_{q<p} round_up(n_q, 16)
 *    of a flat per-rank buffer of S = sum_p round_up(n_p, 16) elements.  The mixed
 *    float8 all-gather slot uses byte offsets boff_p = sum_{q<p} round_up(n_q*e_q, 16)
 *    with e = 1 (e4m3fn, fp8-eligible params) or 2 (bf16).
 */
#ifndef FSDP_B200_H
#define FSDP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSDP_B200_ABI_VERSION 2   /* 2: FSDP_PROF_REPLICA_GATHER (profile arrays of 16) */
#define FSDP_MAX_NDIM 8
#define FSDP_UNIQUE_ID_BYTES 128

typedef enum {
  FSDP_OK = 0,
  FSDP_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, bad enum, out-of-range index          */
  FSDP_ERR_SHAPE = 2,            /* 0-dim param, ranks disagree on the layout   */
  FSDP_ERR_DTYPE = 3,            /* dtype combination not supported                      */
  FSDP_ERR_STATE = 4,            /* call out of order (e.g. unsharded_param before wait) */
  FSDP_ERR_OUT_OF_MEMORY = 5,
  FSDP_ERR_CUDA = 6,
  FSDP_ERR_NCCL = 7,
  FSDP_ERR_TIMEOUT = 8,
  FSDP_ERR_NONFINITE = 9,        /* non-finite fp8 amax                     */
  FSDP_ERR_UNAVAILABLE = 10      /* feature not available in this build / mesh           */
} fsdp_status_t;

typedef enum {
  FSDP_FLOAT32 = 0,
  FSDP_BFLOAT16 = 1,
  FSDP_FLOAT8_E4M3FN = 2
} fsdp_dtype_t;

typedef struct fsdp_mesh fsdp_mesh_t;   /* 1-D data-parallel group: NCCL comms, streams */
typedef struct fsdp_layer fsdp_layer_t; /* one FSDP unit (TransformerBlock or root)     */

/* One parameter of an FSDP unit: its full (unsharded) shape and whether it takes part
 * in the Float8 all-gather ("applied selectively to linear layers"). */
typedef struct {
  int32_t ndim;                  /* 1..FSDP_MAX_NDIM; 0-dim -> FSDP_ERR_SHAPE */
  int32_t fp8_eligible;          /* 0/1 */
  int64_t shape[FSDP_MAX_NDIM];  /* shape[0] may be 0 or < world_size */
} fsdp_param_desc_t;

/* Shard(0) metadata of one parameter on one rank (all in elements unless noted). */
typedef struct {
  int64_t dim0;            /* shape[0]                                    */
  int64_t rest;            /* product of shape[1:]                        */
  int64_t chunk_rows;      /* c = ceil(dim0 / W)                          */
  int64_t row_begin;       /* min(r*c, dim0)                              */
  int64_t row_count;       /* rows owned by this rank (may be 0)          */
  int64_t padded_numel;    /* n = c * rest                                */
  int64_t elem_offset;     /* off_p in the flat fp32/bf16 layouts         */
  int64_t fp8_byte_offset; /* boff_p in the mixed float8 all-gather slot  */
} fsdp_param_meta_t;

/* Per-kernel device time accumulated while profiling is on (CUDA events recorded on
 * the stream each kernel is launched on). */
typedef enum {
  FSDP_PROF_COPY_IN = 0,     /* K2/K3 unshard copy-in (bf16 or float8 cast)   */
  FSDP_PROF_ALL_GATHER = 1,  /* NCCL all-gather                               */
  FSDP_PROF_COPY_OUT = 2,    /* K4 unshard copy-out                           */
  FSDP_PROF_RS_COPY_IN = 3,  /* K5 grad chunk-cat + fp32 cast + divide by W   */
  FSDP_PROF_REDUCE_SCATTER = 4,
  FSDP_PROF_RS_COPY_OUT = 5, /* K6 accumulate / widen                          */
  FSDP_PROF_AMAX = 6,        /* K1                                            */
  FSDP_PROF_SCALE = 7,       /* K1b                                           */
  FSDP_PROF_ALL_REDUCE = 8,  /* NCCL all-reduce(max) of the amaxes            */
  FSDP_PROF_UNSHARD_PUSH = 9,  /* P2P: fused copy-in + all-gather + copy-out   */
  FSDP_PROF_RS_PULL = 10,      /* P2P: fused chunk + /W + reduce + copy-out    */
  FSDP_PROF_STAGE_GRADS = 11,  /* P2P: caller grads -> symmetric staging       */
  FSDP_PROF_HANDSHAKE = 12,    /* P2P: cross-GPU ready/done flag kernels       */
  FSDP_PROF_RS_SCATTER = 13,   /* P2P store RS: own grad rows -> peers' receive buffers (NVLink) */
  FSDP_PROF_RS_REDUCE = 14,    /* P2P store RS: local ascending-rank reduce of the receive buffer */
  FSDP_PROF_REPLICA_GATHER = 15, /* HSDP two-phase RS: finished pieces from the replicas -> grad */
  FSDP_PROF_NUM = 16
} fsdp_prof_kind_t;

/* How the collectives of a mesh run.
 *  FSDP_ALGO_NCCL: copy-in kernel -> ncclAllGather -> copy-out kernel; chunk-cat kernel ->
 *                  ncclReduceScatter (fp32).
 *  FSDP_ALGO_P2P:  symmetric buffers mapped with CUDA IPC across the ranks' GPUs (NVLink /
 *                  NVSwitch); the unshard is ONE push kernel (cast + store into every rank's
 *                  unsharded tensors); the reduce-scatter is one store-scatter kernel (every
 *                  rank's rows into its owner's receive buffer) plus a local reduce, or one
 *                  pull kernel (read every rank's bf16 grad rows) — fsdp_mesh_set_p2p_rs —
 *                  both /W and summing in ascending rank order in fp32; every data kernel is
 *                  bracketed by single-CTA flag handshakes.  Requires W <= 8 GPUs with peer
 *                  access; identical results up to the reduce-scatter summation order (P2P:
 *                  ascending rank, deterministic). */
typedef enum { FSDP_ALGO_NCCL = 0, FSDP_ALGO_P2P = 1 } fsdp_algo_t;

typedef struct {
  int64_t launches[FSDP_PROF_NUM];
  double total_ms[FSDP_PROF_NUM];
  int64_t bytes[FSDP_PROF_NUM];  /* algorithmic HBM bytes of those launches */
} fsdp_profile_t;

/* ---------------------------------------------------------------- generic */
int32_t fsdp_abi_version(void);
const char* fsdp_last_error(void);           /* thread-local; "" if none */
const char* fsdp_status_string(fsdp_status_t s);

/* Host-only Shard(0) layout of one unit for (world_size, rank); needs no GPU.
 * out_metas: caller array of n_params entries.  out_hash: 64-bit FNV-1a hash of
 * (W, every desc) — identical on all ranks iff they agree on the unit (the check
 * fsdp_shard performs, "shape mismatch across members").  Any out_* may be NULL. */
fsdp_status_t fsdp_layout_compute(int32_t n_params, const fsdp_param_desc_t* descs,
                                  int32_t world_size, int32_t rank,
                                  fsdp_param_meta_t* out_metas, int64_t* out_S,
                                  int64_t* out_S_bytes_fp8, uint64_t* out_hash);

/* ---------------------------------------------------------------- mesh */
/* Rank 0 calls this and broadcasts the bytes (the Python binding uses the
 * torch.distributed process group for that, its only torch.distributed use). */
fsdp_status_t fsdp_get_unique_id(uint8_t id[FSDP_UNIQUE_ID_BYTES]);

/* Collective over the W ranks: creates two NCCL communicators (all-gather, and
 * reduce-scatter/all-reduce, so unshard of layer i-1 overlaps the reduce-scatter of
 * layer i) plus internal high-priority streams on `cuda_device`.  world_size = the
 * data-parallel shard degree (all ranks by default). */
fsdp_status_t fsdp_mesh_init(const uint8_t id[FSDP_UNIQUE_ID_BYTES], int32_t world_size,
                             int32_t rank, int32_t cuda_device, fsdp_mesh_t** out);

/* A P2P mesh with no NCCL communicator: the few host-side collective steps the library
 * needs (CUDA IPC handle exchange of the symmetric buffers, the layout-hash check, barriers
 * before frees) go through the caller's host all-gather `fn`: send = `bytes` host bytes of
 * this rank, recv = world_size * bytes, rank-major over the whole world; returns 0 on
 * success (e.g. torch.distributed over gloo).  Every device-side step is the P2P path:
 * push unshard, pull / store reduce-scatter, the fp8 amax all-reduce (a P2P max over
 * symmetric memory), HSDP's world reduce-scatter (shard_size < world_size; 0 = all ranks).
 * The ranks may share a GPU (CUDA IPC works between processes on one device), so the
 * cross-process protocol — IPC-mapped arenas, device-epoch handshakes, timeouts — runs
 * where NCCL (one rank per GPU) cannot.  FSDP_ERR_UNAVAILABLE if some rank cannot map
 * every peer (or, with shard_size < world_size, the world); fsdp_mesh_set_algo(NCCL) is
 * unavailable on it.  `fn` and `ctx` must stay valid until fsdp_mesh_destroy returns. */
typedef int32_t (*fsdp_host_allgather_fn)(const void* send, void* recv, int64_t bytes, void* ctx);
fsdp_status_t fsdp_mesh_init_hostcoll(int32_t world_size, int32_t rank, int32_t shard_size, int32_t cuda_device,
                                      fsdp_host_allgather_fn fn, void* ctx, fsdp_mesh_t** out);

/* A mesh without communicators: the layout is that of rank `rank` of `world_size`,
 * the fsdp_stage_* entry points work, the collective calls work only when
 * world_size == 1 (identity collectives) and return FSDP_ERR_UNAVAILABLE otherwise.
 * Used to test every kernel at any W on one GPU. */
fsdp_status_t fsdp_mesh_init_local(int32_t world_size, int32_t rank, int32_t cuda_device,
                                   fsdp_mesh_t** out);

/* HSDP (hybrid sharded data parallel, P:472-478 appendix:hsdp): a 2-D mesh of world_size =
 * replicate_size x shard_size ranks, replica dimension outer: rank g is shard rank
 * g % shard_size of replica g / shard_size (R15).  Parameters are Shard(0) over
 * the shard group (every layout call uses shard_size as W and the shard rank as rank);
 * fsdp_unshard all-gathers within the shard group; fsdp_reduce_scatter_grads divides by
 * world_size (mean over all ranks), reduce-scatters within the shard group
 * and all-reduces (sum, fp32, NCCL) across the replica group ("the addition of backward
 * gradient allreduce across replica groups").  Collective over all world_size
 * ranks; shard_size must divide world_size; shard_size == world_size is plain FSDP.
 * One NVSwitch domain (world_size <= 8, every rank maps every rank's memory, checked
 * collectively here): the reduce-scatter is a pull over the world instead (two-phase by
 * default, fsdp_stage_hsdp_piece_pull / _replica_gather: each replica computes 1/R of the
 * shard, then the replicas exchange the finished fp32 pieces) — each element is the sum of
 * that shard row over all world_size ranks' grads in the same nested
 * order (shard ranks ascending within a replica, then the replica partials ascending, fp32:
 * the oracle's HsdpWorld 'order', bit for bit) with no serial replica all-reduce, and
 * fsdp_full_grad_buffer maps its zero-copy grad buffers over the whole world.
 * FSDP_B200_HSDP_P2P=0 (at init) or fsdp_mesh_set_algo(FSDP_ALGO_NCCL) keeps the
 * reduce-scatter + NCCL all-reduce pair; fsdp_mesh_get_hsdp_rs tells which runs. */
fsdp_status_t fsdp_mesh_init_hsdp(const uint8_t id[FSDP_UNIQUE_ID_BYTES], int32_t world_size,
                                  int32_t rank, int32_t shard_size, int32_t cuda_device,
                                  fsdp_mesh_t** out);
/* replicate_size and this rank's replica index (1 and 0 for a 1-D mesh). */
fsdp_status_t fsdp_mesh_info_hsdp(const fsdp_mesh_t* mesh, int32_t* replicate_size,
                                  int32_t* replica_index);
/* *world_pull: 0 = shard-group reduce-scatter + NCCL all-reduce, 1 = the one-phase world
 * pull above, 2 = the two-phase world reduce-scatter (pieces + replica gather, default). */
fsdp_status_t fsdp_mesh_get_hsdp_rs(const fsdp_mesh_t* mesh, int32_t* world_pull);

/* Destroys the mesh (synchronizes its streams, frees its pools, destroys the comms).
 * All layers of the mesh must have been destroyed. */
fsdp_status_t fsdp_mesh_destroy(fsdp_mesh_t* mesh);
fsdp_status_t fsdp_mesh_info(const fsdp_mesh_t* mesh, int32_t* world_size, int32_t* rank,
                             int32_t* cuda_device);
/* Device memory the mesh holds, in bytes (SURVEY §8(e) sizing at W): out[0] symmetric
 * buffers this rank allocated (flags, P2P arenas and grad staging / receive slots, zero-copy
 * grad buffers); out[1] the peers' copies of them mapped into this process over CUDA IPC
 * (address space only: the peers' HBM); out[2] pooled NCCL-mode / W=1 buffers; out[3] the
 * layers' fp32 shards and sharded grads (+ non-symmetric grad buffers). */
fsdp_status_t fsdp_mesh_memory(const fsdp_mesh_t* mesh, int64_t out[4]);

/* Selects the collective algorithm (fsdp_algo_t).  Collective: every rank must make the
 * same call at the same point, with no layer unsharded / reduce-scatter pending.  The
 * default after fsdp_mesh_init is FSDP_ALGO_P2P when W > 1, W <= 8 and every rank could
 * map its peers' buffers (environment FSDP_B200_ALGO=nccl|p2p overrides), else NCCL.
 * FSDP_ERR_UNAVAILABLE if P2P is requested but not possible.  On an HSDP mesh the choice
 * also selects the reduce-scatter (P2P: the world pull when available); with shard_size 1
 * P2P only switches that on (the unshard is local). */
fsdp_status_t fsdp_mesh_set_algo(fsdp_mesh_t* mesh, int32_t algo);
fsdp_status_t fsdp_mesh_get_algo(const fsdp_mesh_t* mesh, int32_t* algo);

/* How FSDP_ALGO_P2P reduce-scatters (fsdp_p2p_rs_t; same result bits either way: this
 * rank's rows, sum over ranks q = 0..W-1 ascending of fp32(g_q) / W in fp32):
 *  FSDP_P2P_RS_PULL:  every rank stages its full grads into its symmetric staging buffer (or
 *                     writes them into fsdp_full_grad_buffer) and pulls its rows from all
 *                     ranks' staging over NVLink (loads);
 *  FSDP_P2P_RS_STORE: every rank stores each peer's rows of its own grads (read locally, so no
 *                     staging copy for any caller buffer) into that peer's symmetric receive
 *                     buffer over NVLink (stores), then reduces its received rows locally on a
 *                     second stream, overlapping the next unit's transfer.
 *  FSDP_P2P_RS_AUTO:  PULL when the layer has zero-copy grad buffers (fsdp_full_grad_buffer,
 *                     created collectively, so every rank decides alike) and W == 2 or the
 *                     unit moves < 64 MB of bus bytes; else STORE — the faster one on 2 and 4
 *                     B200s.
 * Collective (same call on every rank, nothing pending).  Default: FSDP_P2P_RS_AUTO
 * (environment FSDP_B200_P2P_RS=pull|store|auto overrides). */
typedef enum { FSDP_P2P_RS_PULL = 0, FSDP_P2P_RS_STORE = 1, FSDP_P2P_RS_AUTO = 2 } fsdp_p2p_rs_t;
fsdp_status_t fsdp_mesh_set_p2p_rs(fsdp_mesh_t* mesh, int32_t mode);
fsdp_status_t fsdp_mesh_get_p2p_rs(const fsdp_mesh_t* mesh, int32_t* mode);

/* Waits (host) until every internal stream of the mesh is idle, polling NCCL for
 * asynchronous errors.  Returns FSDP_ERR_NONFINITE if a precompute saw a non-finite
 * amax since the last call (flag is then cleared), FSDP_ERR_NCCL on a NCCL async
 * error, FSDP_ERR_TIMEOUT after timeout_ms (<= 0: no timeout); after NCCL/TIMEOUT the
 * communicators are aborted and the mesh is unusable.  The abort is sticky: every later
 * call on the mesh (this one included) returns the FIRST failure's status and message,
 * whichever call (wait_* or this one) reported it first. */
fsdp_status_t fsdp_mesh_synchronize(fsdp_mesh_t* mesh, int64_t timeout_ms);
/* Marks the mesh unusable without any collective step (aborts its NCCL communicators);
 * layers and the mesh can then be destroyed rank-locally.  Use after FSDP_ERR_TIMEOUT /
 * FSDP_ERR_NCCL on any rank.  P2P handshakes give up after FSDP_B200_P2P_TIMEOUT_MS
 * (default 60000) and report FSDP_ERR_TIMEOUT through fsdp_mesh_synchronize. */
fsdp_status_t fsdp_mesh_abort(fsdp_mesh_t* mesh);

/* Profiling: when on, every kernel / collective launch is bracketed by CUDA events on
 * its own stream; fsdp_profile_read synchronizes and returns the totals since the last
 * reset. */
fsdp_status_t fsdp_profile_enable(fsdp_mesh_t* mesh, int32_t on);
fsdp_status_t fsdp_profile_read(fsdp_mesh_t* mesh, fsdp_profile_t* out, int32_t reset);

/* Device-memory allocator of the mesh's bulk buffers (SURVEY.md §8(b) "Ownership": device
 * memory comes from a caller-supplied allocator, which the Python binding wires to the
 * torch caching allocator — "PyTorch for device memory" without the library calling
 * torch).  alloc_fn(ctx, bytes, device, &ptr) returns 0 and a device pointer of at least
 * `bytes` bytes on `device`, 256-byte aligned (else FSDP_ERR_INVALID_ARGUMENT), or non-zero
 * for out of memory (-> FSDP_ERR_OUT_OF_MEMORY); free_fn(ctx, ptr, device) releases it.
 * The library synchronizes the device before calling free_fn, so the block may be reused
 * on any stream at once.  Covered: every layer's fp32 shard and sharded-grad buffers, the
 * NCCL path's all-gather / reduce-scatter pool buffers and the non-symmetric full-grad
 * buffers (fsdp_full_grad_buffer under NCCL) allocated after the call; each buffer is
 * freed through the allocator that made it.  Not covered (stay cudaMalloc / CUDA-IPC
 * exported, library-owned): the P2P path's symmetric buffers (they must be IPC-mappable
 * allocations of their own) and bookkeeping tables (tiles, fp8 registry; < 1 MB per
 * unit).  Both NULL restores cudaMalloc / cudaFree.  Host-synchronous. */
typedef int32_t (*fsdp_alloc_fn)(void* ctx, size_t bytes, int32_t device, void** out_ptr);
typedef void (*fsdp_free_fn)(void* ctx, void* ptr, int32_t device);
fsdp_status_t fsdp_mesh_set_allocator(fsdp_mesh_t* mesh, fsdp_alloc_fn alloc_fn, fsdp_free_fn free_fn,
                                      void* ctx);

/* ---------------------------------------------------------------- shard (a1) */
/* fsdp_shard(params, mesh): synchronous, collective over the mesh (all ranks call it
 * with the same descs, checked by an all-gather of the layout hash -> FSDP_ERR_SHAPE).
 * Copies descs.  full_params[p] (fp32, contiguous, host or device — anything
 * cudaMemcpyDefault accepts — or NULL to leave the shard zero, or full_params == NULL
 * for all) is read once: this rank's rows go to its flat fp32 shard, padding is +0.0.
 * The layer owns: the fp32 shard [S], the fp32 sharded-grad buffer [S], tile tables. */
fsdp_status_t fsdp_shard(fsdp_mesh_t* mesh, int32_t n_params, const fsdp_param_desc_t* descs,
                         const float* const* full_params, fsdp_layer_t** out);
/* Synchronizes the layer's pending work and frees it.  State must not be UNSHARDED. */
fsdp_status_t fsdp_layer_destroy(fsdp_layer_t* layer);
fsdp_status_t fsdp_layer_info(const fsdp_layer_t* layer, int32_t* n_params, int64_t* S,
                              int64_t* S_bytes_fp8);
fsdp_status_t fsdp_param_meta(const fsdp_layer_t* layer, int32_t p, fsdp_param_meta_t* out);
/* Views into the layer-owned fp32 shard (the optimizer's state; valid until destroy):
 * param p's padded shard is (*dev)[0 .. padded_numel), rows [0,row_count) are real. */
fsdp_status_t fsdp_sharded_param(const fsdp_layer_t* layer, int32_t p, float** dev);
fsdp_status_t fsdp_sharded_flat(const fsdp_layer_t* layer, float** dev);

/* ---------------------------------------------------------------- fp8 scales (a2) */
/* precompute_fp8_scales(params): for every fp8-eligible param of the given layers,
 * amax_p = max over ranks and elements of |shard_p| (one K1 launch over all layers,
 * one NCCL all-reduce(max), one K1b launch), s_p = fp32(448 / fp64(max(amax_p,1e-12))).
 * Stream-ordered on `stream`; results readable via fsdp_fp8_scales after work on
 * `stream`.  A non-finite amax sets the mesh's error flag (see fsdp_mesh_synchronize)
 * and leaves s_p = 0 for that param. */
fsdp_status_t fsdp_precompute_fp8_scales(fsdp_mesh_t* mesh, fsdp_layer_t* const* layers,
                                         int32_t n_layers, void* stream);
/* Delayed scaling ("dynamic, delayed, and static"): the same amax
 * pass and all-reduce(max), then per eligible param s_p = fp32(448 / fp64(max(H_p, 1e-12)))
 * where H_p is the max of the param's amax history (the last history_len amaxes,
 * initialised with the first observed amax), and the current amax is pushed into the
 * history after use.  history_len in [1, 64], fixed by the first call.  Static scaling =
 * passing caller scales to fsdp_unshard.
 * Amax fused into the casts (default; FSDP_B200_AMAX_FUSE=0 turns it off): a delayed call
 * arms its layers, and every later fp8 fsdp_unshard of an armed layer folds max |x| of the
 * fp32 elements it casts into the accumulator (no extra HBM pass).  The next delayed call on
 * the same layers then records that amax into the history FIRST and takes the scale after —
 * the same history as recording it after use at the previous call, so the scales are
 * bit-identical — and skips the amax pass over every shard (only the first call, and an
 * armed layer that was not fp8-unsharded since the previous call, run it).  amax_dev then
 * holds the recorded amax: the previous step's.  The unshards of a step must be waited
 * (fsdp_wait_unshard) before the next step's delayed call; a dynamic call disarms. */
fsdp_status_t fsdp_precompute_fp8_scales_delayed(fsdp_mesh_t* mesh, fsdp_layer_t* const* layers,
                                                 int32_t n_layers, int32_t history_len, void* stream);
/* Device arrays of P floats (entries of non-eligible params are 0).  The pointers stay valid
 * until the mesh is destroyed: the mesh's fp8 registry has a fixed capacity (65536 params,
 * environment FSDP_B200_REGISTRY_CAP) and is never reallocated, so views taken here and
 * kernel arguments captured in CUDA graphs never dangle; fsdp_shard returns
 * FSDP_ERR_UNAVAILABLE when the registry is full.  Entries are assigned in fsdp_shard order
 * and recycled only once every layer of the mesh has been destroyed.
 * Deliberate extension of SURVEY §8(b)'s `fsdp_fp8_scales(layer, scales)`: amax_dev (may
 * be NULL) also exposes the all-reduced amax the scales were taken from, so callers and
 * tests can check the scale formula without recomputing the amax. */
fsdp_status_t fsdp_fp8_scales(const fsdp_layer_t* layer, const float** scales_dev,
                              const float** amax_dev);

/* ---------------------------------------------------------------- unshard (a3-a6) */
/* fsdp_unshard / all_gather_params(layer, dtype, fp8_scale): stream-ordered after
 * `compute`.  Acquires an all-gather buffer from the mesh pool (event-guarded, never
 * record_stream), runs copy-in (K2 bf16 / K3 float8, in place into this
 * rank's slot), the all-gather, and copy-out (K4) into per-parameter full tensors.
 * param_dtype: FSDP_BFLOAT16 or FSDP_FLOAT8_E4M3FN (eligible params in
 * e4m3fn with per-tensor scale, others bf16).  fp8_scales_dev: P device floats, or NULL
 * to use the layer's precomputed scales.  State: SHARDED -> UNSHARDING; on a layer that is
 * already unsharded (reshard_after_forward=False, the kept last block) it is a
 * no-op for the same param_dtype and FSDP_ERR_STATE for another. */
fsdp_status_t fsdp_unshard(fsdp_layer_t* layer, fsdp_dtype_t param_dtype,
                           const float* fp8_scales_dev, void* compute);
/* Makes `compute` wait for the unshard.  State: UNSHARDING -> UNSHARDED.
 * Both wait_* calls also report, without synchronizing, what has already failed
 * asynchronously: a P2P handshake that gave up on a peer (FSDP_ERR_TIMEOUT) or a NCCL async
 * error (FSDP_ERR_NCCL); the mesh is then unusable (fsdp_mesh_abort).  A failure that has not
 * happened yet when wait_* is called is reported by a later wait_* or by
 * fsdp_mesh_synchronize, which drains the streams and reports everything. */
fsdp_status_t fsdp_wait_unshard(fsdp_layer_t* layer, void* compute);
/* fsdp_unshard + fsdp_wait_unshard (the name used by BASELINE.json). */
fsdp_status_t fsdp_all_gather_params(fsdp_layer_t* layer, fsdp_dtype_t param_dtype,
                                     const float* fp8_scales_dev, void* compute);
/* Full tensor of param p (shape = desc shape, row-major, contiguous, 256B-aligned);
 * dtype is BF16 or FLOAT8_E4M3FN.  Valid from wait_unshard until reshard.
 * State must be UNSHARDED, else FSDP_ERR_STATE. */
fsdp_status_t fsdp_unsharded_param(const fsdp_layer_t* layer, int32_t p, void** dev,
                                   fsdp_dtype_t* dtype);
/* Releases the unsharded storage: the buffer returns to the pool once the work
 * enqueued on `compute` so far completes (event-guarded).  UNSHARDED -> SHARDED. */
fsdp_status_t fsdp_reshard(fsdp_layer_t* layer, void* compute);

/* ---------------------------------------------------------------- post-backward (a7-a9) */
/* reduce_scatter_grads(layer, reduce_dtype, mean): full_grads_dev[p] = this rank's
 * full gradient of param p (contiguous, desc shape, grad_dtype BF16 or FLOAT32).
 * K5 chunks every grad on dim 0, widens to fp32, divides once by W when mean != 0
 * (P:466), zero-pads, packs rank-major [W][S]; then a reduce-scatter (sum) in
 * reduce_dtype (FLOAT32 default; BFLOAT16: inputs rounded to bf16 after the
 * division) lands this rank's chunk in the layer's fp32 sharded-grad buffer
 * (accumulate != 0: added to it, in fp32).  The caller keeps full_grads alive and
 * unmodified until fsdp_wait_reduce_scatter (deterministic release). */
fsdp_status_t fsdp_reduce_scatter_grads(fsdp_layer_t* layer, const void* const* full_grads_dev,
                                        fsdp_dtype_t grad_dtype, fsdp_dtype_t reduce_dtype,
                                        int32_t mean, int32_t accumulate, void* compute);
fsdp_status_t fsdp_wait_reduce_scatter(fsdp_layer_t* layer, void* compute);
/* Zero-copy gradients: the layer's own full-gradient buffer (all params, grad_dtype, each
 * param contiguous with its desc shape at a 256-byte aligned offset); *dev = param p's
 * tensor.  The buffer is allocated by the first call — symmetric (mapped into every peer)
 * when the mesh can run FSDP_ALGO_P2P, which makes that first call collective, and so is
 * fsdp_layer_destroy of a layer that has one.  When every full_grads[p] given to
 * fsdp_reduce_scatter_grads is this buffer's tensor (on all ranks alike), the P2P path
 * skips the staging copy and peers read the gradients in place.  Valid until destroy;
 * writable again after fsdp_wait_reduce_scatter.  FSDP_ERR_DTYPE if a later call asks
 * for another grad_dtype. */
fsdp_status_t fsdp_full_grad_buffer(fsdp_layer_t* layer, fsdp_dtype_t grad_dtype, int32_t p, void** dev);
/* fp32 sharded grad of param p: (*dev)[0 .. row_count*rest) (views into the layer's
 * grad buffer, same flat layout as the shard).  Deliberate narrowing of SURVEY §8(b)'s
 * `(void** dev, fsdp_dtype_t* dt)`: the sharded grad is always fp32 here (reduce_dtype
 * BFLOAT16 only changes the reduction's rounding, R11, and the result is widened into the
 * fp32 grad), so the pointer is typed and no dtype is returned. */
fsdp_status_t fsdp_sharded_grad(const fsdp_layer_t* layer, int32_t p, float** dev);
fsdp_status_t fsdp_sharded_grad_flat(const fsdp_layer_t* layer, float** dev);
fsdp_status_t fsdp_zero_grad(fsdp_layer_t* layer, void* stream);

/* ---------------------------------------------------------------- stage entry points */
/* One kernel each, no communication, stream-ordered on `stream`; they expose the
 * individual steps (for tests at any W on one GPU and for custom collectives). */
/* K2/K3: this rank's all-gather slot (S*2 bytes for BF16, S_bytes_fp8 for FLOAT8).
 * amax_accum_dev (FLOAT8 only; NULL = none): P floats read and written as fp32 bit patterns,
 * amax_accum[p] = max(amax_accum[p], max |x| over this rank's cast elements of eligible param
 * p) — the delayed-scaling amax fused into the cast (bit-identical to K1). */
fsdp_status_t fsdp_stage_copy_in(const fsdp_layer_t* layer, fsdp_dtype_t param_dtype,
                                 const float* fp8_scales_dev, void* ag_slot_dev, float* amax_accum_dev,
                                 void* stream);
/* K4: from a full rank-major all-gather buffer [W][slot] into per-param full tensors
 * full_out_dev[p] (contiguous, numel = prod(shape) elements of the param's dtype). */
fsdp_status_t fsdp_stage_copy_out(const fsdp_layer_t* layer, fsdp_dtype_t param_dtype,
                                  const void* ag_buffer_dev, void* const* full_out_dev,
                                  void* stream);
/* K1 on one layer: amax_out_dev[p] = max |shard_p| on this rank (0 if not eligible). */
fsdp_status_t fsdp_stage_local_amax(const fsdp_layer_t* layer, float* amax_out_dev, void* stream);
/* K1b: scale_out[p] = eligible ? fp32(448/fp64(max(amax[p],1e-12))) : 0 (non-finite
 * amax -> 0 and the mesh error flag is set). */
fsdp_status_t fsdp_stage_fp8_scale(const fsdp_layer_t* layer, const float* amax_dev,
                                   float* scale_out_dev, void* stream);
/* K5: rs_in_dev = [W][S] (FLOAT32 or BFLOAT16 per reduce_dtype). */
fsdp_status_t fsdp_stage_rs_copy_in(const fsdp_layer_t* layer, const void* const* full_grads_dev,
                                    fsdp_dtype_t grad_dtype, fsdp_dtype_t reduce_dtype,
                                    int32_t mean, void* rs_in_dev, void* stream);
/* K6: the layer's fp32 grad buffer [S] = (accumulate ? grad + : ) widen(rs_out_dev[S]). */
fsdp_status_t fsdp_stage_rs_copy_out(fsdp_layer_t* layer, const void* rs_out_dev,
                                     fsdp_dtype_t reduce_dtype, int32_t accumulate, void* stream);

/* ---- the P2P kernels without their handshakes (FSDP_ALGO_P2P) */
/* Unsharded arena layout for param_dtype: byte offset of param p (256-byte aligned) and
 * the arena size.  offsets: caller array of P entries (may be NULL). */
fsdp_status_t fsdp_unsharded_layout(const fsdp_layer_t* layer, fsdp_dtype_t param_dtype,
                                    int64_t* offsets, int64_t* total_bytes);
/* K7 push: casts this rank's rows of every param (bf16, or e4m3fn with fp8_scales_dev[p] for
 * eligible params when param_dtype is FLOAT8) and stores them at their place in each of the
 * W arenas arenas_dev[0..W-1] (any device memory the current device can store to, e.g.
 * peer-mapped; each 16-byte aligned, else FSDP_ERR_INVALID_ARGUMENT — the TMA bulk stores
 * address them relative to their base).  Running it for every rank fills every arena with
 * the full tensors.  amax_accum_dev: as in fsdp_stage_copy_in (the fused amax of the push). */
fsdp_status_t fsdp_stage_unshard_push(const fsdp_layer_t* layer, fsdp_dtype_t param_dtype,
                                      const float* fp8_scales_dev, void* const* arenas_dev,
                                      float* amax_accum_dev, void* stream);
/* Grad staging layout: param p's full grad at element offset elem_offsets[p] (128-aligned). */
fsdp_status_t fsdp_grad_staging_layout(const fsdp_layer_t* layer, int64_t* elem_offsets,
                                       int64_t* total_elems);
/* Copies this rank's full grads into a staging buffer of that layout (grad_dtype elements). */
fsdp_status_t fsdp_stage_grads_to_staging(const fsdp_layer_t* layer, const void* const* full_grads_dev,
                                          fsdp_dtype_t grad_dtype, void* staging_dev, void* stream);
/* K8 pull: for this rank's rows, grad (+)= sum over q = 0..W-1 ascending of
 * fp32(stagings_dev[q]) / W (mean) — bf16 reduce_dtype rounds every term and the sum to bf16.
 * Every staging base must be 16-byte aligned (TMA bulk loads; else FSDP_ERR_INVALID_ARGUMENT). */
fsdp_status_t fsdp_stage_rs_pull(fsdp_layer_t* layer, const void* const* stagings_dev,
                                 fsdp_dtype_t grad_dtype, fsdp_dtype_t reduce_dtype, int32_t mean,
                                 int32_t accumulate, void* stream);
/* HSDP world pull (header of fsdp_mesh_init_hsdp): for this rank's rows (shard rank
 * = the layer's rank, W = its shard group), grad (+)= sum over replicas r = 0..replicate-1
 * ascending of ( sum over shard ranks q = 0..W-1 ascending of fp32(stagings_dev[r*W+q]) /
 * (replicate*W) ), both sums fp32 (the oracle's HsdpWorld 'order').  stagings_dev: one
 * staging per global rank g = r*W + q, laid out as fsdp_grad_staging_layout, 16-byte
 * aligned.  replicate * W <= 8; replicate must equal the mesh's replicate size unless the
 * mesh is 1-D (a local mesh emulating one shard rank). */
fsdp_status_t fsdp_stage_rs_pull_hsdp(fsdp_layer_t* layer, const void* const* stagings_dev, int32_t replicate,
                                      fsdp_dtype_t grad_dtype, fsdp_dtype_t reduce_dtype, int32_t mean,
                                      int32_t accumulate, void* stream);
/* HSDP two-phase reduce-scatter (the default world pull when R W > 3, where it moves fewer
 * bytes; FSDP_B200_HSDP_RS=1 selects the one-phase pull above).  The shard's flat range [0, S) is cut into `replicate` pieces of
 * P = round_up(ceil(S / replicate), 16) elements; piece q is computed by replica q.
 * Phase 1: res_dev[j] (fp32, laid out like the sharded grad, 16-byte aligned) = the nested
 * sum above for every real element j of piece `replica` (other entries untouched).
 * Phase 2: for every real element j of every piece q, grad[j] (+)= res_devs[q][j], where
 * res_devs[q] is replica q's phase-1 buffer (same shard rank).  Together: the world pull's
 * bits with (RW-1) 2 S / R + (R-1) 4 S / R bytes read per rank instead of (RW-1) 2 S. */
fsdp_status_t fsdp_stage_hsdp_piece_pull(fsdp_layer_t* layer, const void* const* stagings_dev, int32_t replicate,
                                         int32_t replica, fsdp_dtype_t grad_dtype, fsdp_dtype_t reduce_dtype,
                                         int32_t mean, float* res_dev, void* stream);
fsdp_status_t fsdp_stage_hsdp_replica_gather(fsdp_layer_t* layer, const float* const* res_devs, int32_t replicate,
                                             int32_t accumulate, void* stream);
/* Store-based reduce-scatter (FSDP_P2P_RS_STORE), sender: for every rank r, this rank's
 * full-grad rows of r's Shard(0) chunk of each param are copied into r's receive buffer
 * recv_dev[r] at slot `rank`: recv_r[(rank * S + off_p) + j] (grad_dtype elements; a receive
 * buffer is W * S elements, every slot laid out like the flat shard).  recv_dev: W pointers
 * the current device can store to (peer-mapped in the real path).  include_self = 0 skips
 * r = rank (the receiver then reads its own rows from its grads, see below). */
fsdp_status_t fsdp_stage_rs_scatter(const fsdp_layer_t* layer, const void* const* full_grads_dev,
                                    fsdp_dtype_t grad_dtype, void* const* recv_dev, int32_t include_self,
                                    void* stream);
/* Store-based reduce-scatter, receiver: for this rank's rows, grad (+)= sum over q = 0..W-1
 * ascending of fp32(x_q) / W (mean): the same arithmetic as the pull.  x_q = recv[q * S +
 * off_p + j]; when own_grads_dev (P pointers, this rank's full grads) is not NULL, x_rank
 * is read from own_grads_dev[p] + row_begin * rest + j instead of slot `rank` (the default
 * P2P path does this: no own-slot copy).  recv_dev and the own grads must be 16-byte aligned,
 * and with own_grads_dev every own-row offset row_begin * rest * grad_size must be a multiple
 * of 16 bytes (else FSDP_ERR_INVALID_ARGUMENT; the P2P path then uses the own slot). */
fsdp_status_t fsdp_stage_rs_recv_reduce(fsdp_layer_t* layer, const void* recv_dev, const void* const* own_grads_dev,
                                        fsdp_dtype_t grad_dtype, fsdp_dtype_t reduce_dtype, int32_t mean,
                                        int32_t accumulate, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FSDP_B200_H */
