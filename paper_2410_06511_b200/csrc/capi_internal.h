// Internal declarations shared by the C-ABI translation units (capi_*.cpp): error
// handling, RAII helpers, buffer pools, symmetric (CUDA IPC) buffers, and the mesh /
// layer objects behind the opaque handles of include/fsdp_b200.h.  Not installed.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "fsdp_b200.h"
#include "kernels.h"
#include "layout.h"
#include "p2p.h"

namespace fsdpc {

using fsdpk::Tile;
using fsdpl::Layout;


extern thread_local std::string g_last_error;

struct Error {
  fsdp_status_t st;
  std::string msg;
};

[[noreturn]] inline void fail(fsdp_status_t st, const std::string& msg) { throw Error{st, msg}; }

#define CUDA_CHECK(x)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      fail(e_ == cudaErrorMemoryAllocation ? FSDP_ERR_OUT_OF_MEMORY : FSDP_ERR_CUDA,         \
           std::string(#x) + ": " + cudaGetErrorString(e_));                                 \
  } while (0)

#define NCCL_CHECK(x)                                                                        \
  do {                                                                                       \
    ncclResult_t r_ = (x);                                                                   \
    if (r_ != ncclSuccess) fail(FSDP_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

template <class F>
fsdp_status_t guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return FSDP_OK;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.st;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return FSDP_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FSDP_ERR_CUDA;
  }
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CUDA_CHECK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Allocator of the bulk device buffers (fsdp_mesh_set_allocator); no callbacks = cudaMalloc.
// Buffers keep a copy of the allocator that made them and are freed through it.
struct Allocator {
  fsdp_alloc_fn alloc_fn = nullptr;
  fsdp_free_fn free_fn = nullptr;
  void* ctx = nullptr;
  int device = 0;
  void* allocate(size_t bytes) const {
    void* p = nullptr;
    if (!alloc_fn) {
      CUDA_CHECK(cudaMalloc(&p, bytes));
      return p;
    }
    if (alloc_fn(ctx, bytes, device, &p) != 0 || !p) fail(FSDP_ERR_OUT_OF_MEMORY, "allocator callback failed");
    if (reinterpret_cast<uintptr_t>(p) & 255) {
      free_fn(ctx, p, device);
      fail(FSDP_ERR_INVALID_ARGUMENT, "allocator callback returned a pointer that is not 256-byte aligned");
    }
    return p;
  }
  void release(void* p) const {   // never throws (destroy paths)
    if (!p) return;
    if (!free_fn) {
      cudaFree(p);
      return;
    }
    cudaDeviceSynchronize();      // a callback free is not stream-ordered against our kernels
    cudaGetLastError();
    free_fn(ctx, p, device);
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  Allocator al;
  void ensure(size_t bytes, const Allocator& with) {
    if (bytes <= cap) return;
    release();
    // +64 B slack: the misaligned 16-byte loads of K4/K5 may touch the aligned block
    // holding the last byte
    al = with;
    p = al.allocate(bytes + 64);
    cap = bytes;
  }
  void release() {
    al.release(p);
    p = nullptr;
    cap = 0;
  }
};

struct DevTiles {
  Tile* d = nullptr;
  int n = 0;
  std::vector<int> first;   // per-param first tile (param-major tables)
  void upload(const std::vector<Tile>& h) {
    release();
    n = (int)h.size();
    if (n) {
      CUDA_CHECK(cudaMalloc(&d, sizeof(Tile) * h.size()));
      CUDA_CHECK(cudaMemcpy(d, h.data(), sizeof(Tile) * h.size(), cudaMemcpyHostToDevice));
    }
  }
  void release() {
    if (d) cudaFree(d);
    d = nullptr;
    n = 0;
  }
};

// CUDA graph capture state of a stream.  Every stream-ordered call is capturable
// (include/fsdp_b200.h "CUDA graphs"): while the caller's stream is capturing, pools pick
// buffers without querying events and never grow, profiling is off, and a pooled buffer's
// release event is waited on only if it was recorded in the same capture.
struct Capture {
  bool on = false;
  unsigned long long id = 0;
};
inline Capture capture_of(cudaStream_t s) {
  Capture c;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(s, &st, &id) == cudaSuccess && st == cudaStreamCaptureStatusActive) {
    c.on = true;
    c.id = id;
  }
  cudaGetLastError();
  return c;
}

struct Slot {             // one pooled buffer set
  DevBuf a, b;            // AG: a = [W][slot] buffer, b = unsharded arena
                          // RS: a = [W][S] reduce-scatter input, b = staging output [S]
  cudaEvent_t free_ev = nullptr;
  bool in_use = false;
  bool ever_used = false;
  uint64_t last_use = 0;
  cudaEvent_t cap_ev = nullptr;        // releases recorded inside a capture (free_ev: eager only)
  unsigned long long ev_capture = 0;   // capture of the last release (0: eager)
};

// `st` waits until a pooled buffer's previous user released it.  Eager releases record
// free_ev; releases inside a capture record cap_ev (an event recorded during a capture
// cannot be waited on outside it).  Inside a capture, a release recorded outside it is
// already complete (capture begins after a device synchronize, as torch.cuda.graph does),
// so only releases from the same capture become graph dependencies.  Eager calls after a
// replay are ordered after the whole graph by the compute-stream event every call waits on.
template <class SlotT>
inline void wait_released(cudaStream_t st, const SlotT* s, const Capture& cap) {
  if (!s->ever_used) return;
  if (cap.on) {
    if (s->ev_capture == cap.id && s->cap_ev) CUDA_CHECK(cudaStreamWaitEvent(st, s->cap_ev, 0));
    return;
  }
  CUDA_CHECK(cudaStreamWaitEvent(st, s->free_ev, 0));
}

struct ProfRec {
  int kind;
  cudaEvent_t a, b;
  int64_t bytes;
};

// A symmetric buffer: same size on every rank, peers' copies mapped with CUDA IPC.
struct SymBuf {
  void* local = nullptr;
  size_t bytes = 0;
  std::vector<void*> peers;   // peers[r] = rank r's buffer in this process (peers[rank] = local)
  int grp = 0;                // the group it is symmetric over: GRP_SHARD or GRP_WORLD (HSDP)
};

// Groups a symmetric buffer / handshake spans: the Shard(0) group (FSDP, and the HSDP
// unshard), or the whole world (the HSDP reduce-scatter pull on one NVSwitch domain).
enum GroupKind { GRP_SHARD = 0, GRP_WORLD = 1 };

// A pooled symmetric slot of the P2P path (unsharded arena, or grad staging).  Slots are
// chosen deterministically (same choice on every rank) and each use bumps the epoch the
// cross-GPU flags are compared against.
struct SymSlot {
  SymBuf buf;
  cudaEvent_t free_ev = nullptr;
  bool in_use = false;
  bool ever_used = false;
  cudaEvent_t cap_ev = nullptr;        // releases recorded inside a capture (see wait_released)
  unsigned long long ev_capture = 0;   // capture of the last release (0: eager)
  int index = 0;                       // flag slot; handshake epochs live on the device
};

constexpr int kFlagSlots = 512;  // flag slots per kind: pooled slots first, then layer grad buffers
constexpr int kAmaxSlot = kFlagSlots - 1;   // the P2P fp8 amax all-reduce's flag slot
constexpr int kPoolSlots = 64;   // max pooled symmetric slots (arenas / staging) per pool
constexpr int kHistMax = 64;     // max delayed-scaling amax history length
constexpr int kRegCapDefault = 65536;   // fp8 registry entries per mesh (FSDP_B200_REGISTRY_CAP)
enum FlagKind { FK_AG_READY = 0, FK_AG_DONE = 1, FK_RS_READY = 2, FK_RS_DONE = 3, FK_NUM = 4 };

enum LayerState { SHARDED = 0, UNSHARDING = 1, UNSHARDED = 2 };


}  // namespace fsdpc

// the opaque handle types of the C ABI are global structs built from the internal types
using namespace fsdpc;  // NOLINT (internal header, included only by capi_*.cpp)

struct fsdp_layer;

struct fsdp_mesh {
  int W = 1, rank = 0, device = 0;   // shard group size / shard rank
  int R = 1, rep = 0;                // HSDP replicate group size / replica index
  bool local = true;
  ncclComm_t comm_ag = nullptr, comm_rs = nullptr;
  ncclComm_t comm_world = nullptr, comm_rep = nullptr;   // HSDP only
  cudaStream_t s_cin = nullptr, s_ag = nullptr, s_cout = nullptr, s_rsc = nullptr, s_rs = nullptr;
  cudaStream_t s_ce = nullptr;     // copy-engine transfers of the unshard (FSDP_B200_CE)
  cudaEvent_t ev_ce = nullptr;     // cast of param p done -> its copies may start (reused per param)
  bool ce = false;                 // P2P transfers by the copy engines (cudaMemcpyAsync over the IPC
                                   // mappings) instead of SM stores; FSDP_B200_CE=1

  fsdpk::LaunchCfg cfg{};
  std::vector<Slot*> ag_slots, rs_slots;
  uint64_t use_seq = 0;
  // fp8 scale registry: one entry per param of every layer (contiguous per layer); fixed
  // capacity, never reallocated (pointers from fsdp_fp8_scales stay valid)
  int reg_size = 0, reg_cap = 0;
  uint32_t* reg_acc = nullptr;
  float* reg_amax = nullptr;
  float* reg_scale = nullptr;
  uint8_t* reg_elig = nullptr;
  float* reg_hist = nullptr;      // delayed scaling: [reg_cap][kHistMax] amax history
  int32_t* reg_pos = nullptr;
  uint8_t* reg_hinit = nullptr;
  int hist_len = 0;               // fixed at the first delayed precompute
  int* d_err = nullptr;              // device view of h_err (mapped pinned host memory)
  volatile int* h_err = nullptr;
  cudaEvent_t ev_pre_call = nullptr, ev_pre_done = nullptr;
  std::vector<fsdp_layer*> layers;
  // precompute cache: layer list -> (amax tiles, finalize index list)
  struct PreSet {
    std::vector<fsdp_layer*> layers;
    DevTiles tiles;
    int32_t* idx = nullptr;
    int nidx = 0;
    int64_t bytes = 0;
  };
  std::vector<PreSet*> presets;
  // profiling
  bool prof = false;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  fsdp_profile_t prof_acc{};
  bool aborted = false;
  fsdp_status_t abort_status = FSDP_ERR_STATE;   // why (sticky: every later call reports it)
  std::string abort_msg = "mesh was aborted by fsdp_mesh_abort";
  // P2P (fused peer-memory) path
  int algo = FSDP_ALGO_NCCL;
  int p2p_rs_mode = FSDP_P2P_RS_AUTO;        // how the P2P reduce-scatter moves data
  int reduce_per_sm = 2;                     // store-RS local reduce CTAs/SM (0: default grid; 2 measured best)
  int gather_per_sm = 0;                     // HSDP replica gather CTAs/SM (0: default grid)
  bool amax_fuse = true;                     // delayed scaling: amax fused into the fp8 casts (FSDP_B200_AMAX_FUSE=0: K1 pass)
  bool store_own_direct = true;              // store RS: own rows read from the caller's grads (FSDP_B200_STORE_OWN=0: own slot)
  bool p2p_ok = false;
  SymBuf flags;                              // uint64 [FK_NUM][kFlagSlots][kMaxRanks]
  SymBuf amax_sym;                           // P2P fp8 amax all-reduce: uint32 [reg_cap] per rank
  // host-collective mesh (fsdp_mesh_init_hostcoll): no NCCL; host steps via the callback
  fsdp_host_allgather_fn hc_fn = nullptr;
  void* hc_ctx = nullptr;
  // HSDP on one NVSwitch domain (R > 1, R * W <= 8, every rank maps every rank): the
  // reduce-scatter pulls this rank's shard rows from all R * W ranks and sums them in the
  // oracle's nested order (shard ranks, then replicas) — no separate replica all-reduce.
  // World-group symmetric memory: its own flags, epochs, staging pool.
  bool hsdp_p2p = false;                     // capability (collective check at init)
  bool hsdp_rs_p2p = false;                  // in use (FSDP_B200_HSDP_P2P=0 / set_algo(NCCL): off)
  bool hsdp_two_phase = true;                // world RS of 1/R pieces + replica gather when R W > 3 (FSDP_B200_HSDP_RS=1: one pull)
  SymBuf wflags;
  std::vector<SymSlot*> p2p_wrs;             // world grad staging
  unsigned long long* d_wepochs = nullptr;
  std::vector<SymSlot*> p2p_ag, p2p_rs;      // unsharded arenas, grad staging
  uint64_t rs_rr = 0;                        // round robin over staging slots
  int gbuf_seq = 0;                          // flag slots of layer grad buffers: kPoolSlots + seq
  unsigned long long p2p_timeout_ns = 60ull * 1000 * 1000 * 1000;   // handshake spin bound
  int* d_barrier = nullptr;
  // handshake epochs [FK_NUM][kFlagSlots], advanced by the handshake kernels themselves so
  // that a captured CUDA graph signals fresh epochs on every replay
  unsigned long long* d_epochs = nullptr;
  Allocator allocator;                       // bulk buffers (fsdp_mesh_set_allocator)
};

struct fsdp_layer {
  fsdp_mesh* mesh = nullptr;
  int P = 0;
  std::vector<fsdp_param_desc_t> descs;
  Layout L;
  float* shard = nullptr;
  float* grad = nullptr;
  int reg_base = 0;
  int32_t* d_idx_local = nullptr;   // 0..P-1 (stage fp8 scale)
  DevTiles t_cin_fp8, t_cout_bf16, t_cout_fp8, t_rsin;
  DevTiles t_amax_stage;             // fsdp_stage_local_amax (lazily built)
  int64_t bytes_cin_fp8 = 0, bytes_cout_bf16 = 0, bytes_cout_fp8 = 0;
  int64_t grad_numel_total = 0;
  // unshard state
  int state = SHARDED;
  Slot* slot = nullptr;
  fsdp_dtype_t ushard_dtype = FSDP_BFLOAT16;
  cudaEvent_t ev_call = nullptr, ev_cin = nullptr, ev_ag = nullptr, ev_done = nullptr;
  // reduce-scatter state
  bool rs_pending = false;
  cudaEvent_t ev_rcall = nullptr, ev_k5 = nullptr, ev_rs_done = nullptr;
  // P2P path
  DevTiles t_push_bf16, t_push_fp8, t_pull, t_stage_bf16, t_stage_fp32;
  DevTiles t_scatter_bf16, t_scatter_fp32, t_recv;   // store-based reduce-scatter
  // store RS with the own rows read from the caller's grads: scatter tables without the
  // own chunk, receiver tiles with the own-row source offsets (layout.h)
  DevTiles t_scatter_peers_bf16, t_scatter_peers_fp32, t_recv_own;
  bool own_ok_bf16 = false, own_ok_fp32 = false;   // own-row offsets 16-byte aligned
  // delayed fp8 scaling with the amax fused into the casts: armed by a delayed precompute
  // (the fp8 unshards then fold max |x| into the registry accumulator), pushed = an armed fp8
  // unshard ran since the last precompute; t_amax_reg: K1 tiles of this layer alone
  // (registry indices), the stand-in for an armed layer that was not unsharded in a step
  bool amax_armed = false, amax_pushed = false;
  std::vector<int> push_tile_off_bf16, push_tile_off_fp8;   // first push tile of param p (P+1 entries)
  DevTiles t_amax_reg;
  std::vector<int64_t> stg_off_el;   // full-grad staging: param p at element offset (128-aligned)
  int64_t stg_elems = 0;
  int64_t push_bytes_bf16 = 0, push_bytes_fp8 = 0, pull_elems = 0;
  int64_t scatter_elems = 0;         // store RS: elements this rank stores into other ranks
  bool arena_is_flat_bf16 = false;   // every param's bf16 arena offset == 2 * off_p (W=1: K2 casts into it)
  int64_t local_push_bf16 = 0, local_push_fp8 = 0;
  SymSlot* p2p_slot = nullptr;       // arena of the current P2P unshard
  SymSlot* gbuf = nullptr;           // zero-copy full-grad buffer (fsdp_full_grad_buffer)
  bool gbuf_sym = false;
  fsdp_dtype_t gbuf_dtype = FSDP_BFLOAT16;
  void* arena_base = nullptr;        // base of the unsharded tensors (either path)
  // HSDP two-phase reduce-scatter (built on first use for a replicate size): t_piece[q] =
  // the pull tiles of piece q of the shard, t_gather = all of them with tile.pad = q
  int piece_R = 0;
  std::vector<DevTiles> t_piece;
  DevTiles t_gather;
  Allocator al;                      // made shard / grad / non-symmetric gbuf (mesh's at shard time)
};


namespace fsdpc {

// ---- helpers (capi_util.cpp)
cudaEvent_t new_event(bool timing = false);
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
void prof_collect(fsdp_mesh* m);
Slot* acquire_slot(fsdp_mesh* m, std::vector<Slot*>& pool, size_t a_bytes, size_t b_bytes, int min_slots,
                   const Capture& cap);
void release_slot(Slot* s, cudaStream_t last_user, const Capture& cap);
void check_mesh(const fsdp_mesh* m);
void check_layer(const fsdp_layer* l);
void check_param(const fsdp_layer* l, int p);
bool comm_ready(const fsdp_mesh* m);
void registry_init(fsdp_mesh* m);
int registry_reserve(fsdp_mesh* m, int n);
void registry_ensure_hist(fsdp_mesh* m);
void clear_presets(fsdp_mesh* m);
int64_t dtype_size(fsdp_dtype_t d);
// a group: its communicator, size and this rank's index in it
struct Group {
  ncclComm_t comm;
  int W, rank;
};
Group group_of(const fsdp_mesh* m, int grp);
// All-gather of `bytes` host bytes per group rank into recv[G.W][bytes] (group rank order):
// the host callback (host-collective mesh) or NCCL on the device (host-synchronous).
void group_allgather_host(fsdp_mesh* m, int grp, const void* send, void* recv, size_t bytes);
// NCCL communicators exist (a NCCL mesh with W > 1 or HSDP); false for local and
// host-collective meshes
bool nccl_ok(const fsdp_mesh* m);
// fp8 amax all-reduce(max) of reg_acc[0, n) over the shard group through symmetric memory
// (P2P meshes): copy into amax_sym, ready handshake, max over every rank's copy, done
// handshake; stream-ordered on `st`, graph-capturable.
void p2p_amax_allreduce(fsdp_mesh* m, int n, cudaStream_t st);
void mesh_barrier(fsdp_mesh* m, int grp = GRP_SHARD);
bool mesh_all_ok(fsdp_mesh* m, bool ok, int grp = GRP_SHARD);
void sym_free_local(fsdp_mesh* m, SymBuf& b);
void sym_free(fsdp_mesh* m, SymBuf& b);   // collective over b.grp
bool sym_alloc(fsdp_mesh* m, SymBuf& b, size_t bytes, int grp = GRP_SHARD);
fsdpp::FlagPtrs flag_remote(fsdp_mesh* m, int kind, int slot, int grp = GRP_SHARD);
unsigned long long* flag_local(fsdp_mesh* m, int kind, int slot, int grp = GRP_SHARD);
unsigned long long* epoch_ctr(fsdp_mesh* m, int kind, int slot, int grp = GRP_SHARD);
SymSlot* acquire_sym_slot(fsdp_mesh* m, std::vector<SymSlot*>& pool, size_t bytes, int prefer, const Capture& cap,
                          int grp = GRP_SHARD);
void release_sym_slot(SymSlot* s, cudaStream_t last_user, const Capture& cap);
fsdpp::PeerPtrs peer_ptrs(const fsdp_mesh* m, const SymBuf& b);
void p2p_teardown(fsdp_mesh* m);
void launch_copy_out_all(fsdp_layer* l, bool fp8, const void* ag, void* const* outs, cudaStream_t st);
void launch_rs_copy_in_all(fsdp_layer* l, const void* const* grads, bool grad_bf16, void* rs_in, bool out_bf16,
                           bool mean, cudaStream_t st);
int64_t cin_bytes(const fsdp_layer* l, bool fp8);
int64_t slot_bytes(const fsdp_layer* l, bool fp8);
void poll_async_errors(fsdp_mesh* m);
// One fsdp_reduce_scatter_grads call (capi_layer.cpp validates it) and its mechanisms
// (capi_rs.cpp): each enqueues the work, records l->ev_rs_done, sets l->rs_pending.
struct RsCall {
  fsdp_layer* l;
  fsdp_mesh* m;
  const void* const* grads;
  fsdp_dtype_t gd;
  bool obf;            // reduce_dtype BFLOAT16 (R11)
  int64_t osz, S;      // reduce element size, flat shard length
  bool hsdp;           // R > 1
  int divisor;         // W * R (mean over every rank)
  bool via_temp;       // HSDP + accumulate on the NCCL pair: through a temp T
  int32_t mean, accumulate;
  cudaStream_t cs;     // the caller's compute stream
  Capture cap;
  void replica_all_reduce(float* buf, cudaStream_t st) const;   // fp32 ncclAllReduce across replicas
  void add_temp_into_grad(const float* T, cudaStream_t st) const;
};
void rs_hsdp_world(const RsCall& c);
void rs_p2p_store(const RsCall& c);
void rs_p2p_pull(const RsCall& c);
void rs_nccl(const RsCall& c);
// HSDP two-phase reduce-scatter: builds l->t_piece / l->t_gather for R pieces (once per R).
void ensure_pieces(fsdp_layer* l, int R);
// byte offset of the fp32 result region [S] in a world RS buffer (after the grad staging)
inline int64_t hsdp_res_offset(const fsdp_layer* l, int64_t gsz) {
  return ((std::max<int64_t>(l->stg_elems, 128) * gsz + 255) / 256) * 256;
}
// Marks the mesh aborted with a sticky reason and throws it (later calls re-report it).
[[noreturn]] void abort_mesh(fsdp_mesh* m, fsdp_status_t st, const std::string& msg);
// Copy-engine unshard (FSDP_B200_CE): cast this rank's rows into arenas.p[rank] one param at
// a time (push kernel, local arena only) on `st`; after each param's cast the copy engines
// send its rows to every other rank's arena (cudaMemcpyAsync on m->s_ce, peers in the order
// rank+1, rank+2, ...); `st` then waits for the copies.
void ce_unshard(fsdp_layer* l, bool fp8, const float* scales, const fsdpp::PeerPtrs& arenas, cudaStream_t st,
                uint32_t* amax_acc);
// Copy-engine store-scatter: this rank's rows of every other rank r's chunk (and of its own
// when include_self) -> recvs.p[r] at slot `rank` (one cudaMemcpyAsync per rank and param, on
// `st`, ranks in the order rank+1, rank+2, ...).
void ce_scatter(fsdp_layer* l, const void* const* grads, int64_t gsz, const fsdpp::PeerPtrs& recvs, cudaStream_t st,
                bool include_self);   // wait_*: report device timeouts / NCCL async errors seen so far
void do_copy_in(fsdp_layer* l, bool fp8, const float* scales, void* dst, cudaStream_t st,
                uint32_t* amax_acc = nullptr);
void validate_grads(const fsdp_layer* l, const void* const* grads, fsdp_dtype_t gd, fsdp_dtype_t rd);
// TMA bulk copies and 16-byte vector accesses address caller buffers relative to their base:
// the base must be 16-byte aligned (FSDP_ERR_INVALID_ARGUMENT otherwise, before any launch)
inline void check_align16(const void* p, const char* what) {
  if (reinterpret_cast<uintptr_t>(p) & 15u) fail(FSDP_ERR_INVALID_ARGUMENT, std::string(what) + " is not 16-byte aligned");
}


// ---- profiling helpers
struct ProfScope {
  fsdp_mesh* m;
  int kind;
  cudaStream_t st;
  int64_t bytes;
  cudaEvent_t a = nullptr;
  ProfScope(fsdp_mesh* m_, int k, cudaStream_t s, int64_t b) : m(m_), kind(k), st(s), bytes(b) {
    if (!m->prof || capture_of(st).on) return;   // no timing events inside a CUDA graph
    a = take();
    CUDA_CHECK(cudaEventRecord(a, st));
  }
  cudaEvent_t take() {
    if (!m->ev_pool.empty()) {
      cudaEvent_t e = m->ev_pool.back();
      m->ev_pool.pop_back();
      return e;
    }
    return new_event(true);
  }
  void done() {
    if (!m->prof || !a) return;
    cudaEvent_t b = take();
    CUDA_CHECK(cudaEventRecord(b, st));
    m->prof_recs.push_back(ProfRec{kind, a, b, bytes});
    a = nullptr;
  }
};



}  // namespace fsdpc
