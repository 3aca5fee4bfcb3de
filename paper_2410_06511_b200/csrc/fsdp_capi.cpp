// C-ABI implementation (include/fsdp_b200.h): mesh (NCCL communicators + streams +
// buffer pools), layers (fp32 shard, sharded grad, tile tables), and the stream-ordered
// unshard / reshard / reduce-scatter / fp8-precompute calls.
//
// Stream topology per mesh (all high priority, non-blocking):
//   s_cin  : K2/K3 copy-in                       (unshard of layer i+1 runs here while
//   s_ag   : NCCL all-gather on comm_ag           the all-gather of layer i is on s_ag
//   s_cout : K4 copy-out                          and its copy-out on s_cout)
//   s_rsc  : K5 RS copy-in
//   s_rs   : NCCL reduce-scatter / all-reduce(max) on comm_rs, then K6, K1, K1b
// Two communicators let the all-gather of layer i-1 overlap the reduce-scatter of layer
// i in backward.  Buffer reuse is guarded by CUDA events recorded on the consuming
// stream (never cudaStreamAddCallback/record_stream), so memory is released
// deterministically.
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

using fsdpk::Tile;
using fsdpl::Layout;

namespace {

thread_local std::string g_last_error;

struct Error {
  fsdp_status_t st;
  std::string msg;
};

[[noreturn]] void fail(fsdp_status_t st, const std::string& msg) { throw Error{st, msg}; }

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

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) CUDA_CHECK(cudaFree(p));
    p = nullptr;
    cap = 0;
    // +64 B slack: the misaligned 16-byte loads of K4/K5 may touch the aligned block
    // holding the last byte
    CUDA_CHECK(cudaMalloc(&p, bytes + 64));
    cap = bytes;
  }
  void release() {
    if (p) cudaFree(p);
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

struct Slot {             // one pooled buffer set
  DevBuf a, b;            // AG: a = [W][slot] buffer, b = unsharded arena
                          // RS: a = [W][S] reduce-scatter input, b = staging output [S]
  cudaEvent_t free_ev = nullptr;
  bool in_use = false;
  bool ever_used = false;
  uint64_t last_use = 0;
};

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
};

// A pooled symmetric slot of the P2P path (unsharded arena, or grad staging).  Slots are
// chosen deterministically (same choice on every rank) and each use bumps the epoch the
// cross-GPU flags are compared against.
struct SymSlot {
  SymBuf buf;
  cudaEvent_t free_ev = nullptr;
  bool in_use = false;
  bool ever_used = false;
  uint64_t epoch = 0;
  int index = 0;
};

constexpr int kFlagSlots = 512;  // flag slots per kind: pooled slots first, then layer grad buffers
constexpr int kPoolSlots = 64;   // max pooled symmetric slots (arenas / staging) per pool
constexpr int kHistMax = 64;     // max delayed-scaling amax history length
enum FlagKind { FK_AG_READY = 0, FK_AG_DONE = 1, FK_RS_READY = 2, FK_RS_DONE = 3, FK_NUM = 4 };

enum LayerState { SHARDED = 0, UNSHARDING = 1, UNSHARDED = 2 };

}  // namespace

struct fsdp_layer;

struct fsdp_mesh {
  int W = 1, rank = 0, device = 0;   // shard group size / shard rank
  int R = 1, rep = 0;                // HSDP replicate group size / replica index
  bool local = true;
  ncclComm_t comm_ag = nullptr, comm_rs = nullptr;
  ncclComm_t comm_world = nullptr, comm_rep = nullptr;   // HSDP only
  cudaStream_t s_cin = nullptr, s_ag = nullptr, s_cout = nullptr, s_rsc = nullptr, s_rs = nullptr;
  fsdpk::LaunchCfg cfg{};
  std::vector<Slot*> ag_slots, rs_slots;
  uint64_t use_seq = 0;
  // fp8 scale registry: one entry per param of every layer (contiguous per layer)
  int reg_size = 0, reg_cap = 0;
  uint32_t* reg_acc = nullptr;
  float* reg_amax = nullptr;
  float* reg_scale = nullptr;
  uint8_t* reg_elig = nullptr;
  float* reg_hist = nullptr;      // delayed scaling: [reg_cap][kHistMax] amax history
  int32_t* reg_pos = nullptr;
  uint8_t* reg_hinit = nullptr;
  int hist_len = 0;               // fixed at the first delayed precompute
  int* d_err = nullptr;
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
  // P2P (fused peer-memory) path
  int algo = FSDP_ALGO_NCCL;
  bool p2p_ok = false;
  SymBuf flags;                              // uint64 [FK_NUM][kFlagSlots][kMaxRanks]
  std::vector<SymSlot*> p2p_ag, p2p_rs;      // unsharded arenas, grad staging
  uint64_t rs_rr = 0;                        // round robin over staging slots
  int gbuf_seq = 0;                          // flag slots of layer grad buffers: kPoolSlots + seq
  unsigned long long p2p_timeout_ns = 60ull * 1000 * 1000 * 1000;   // handshake spin bound
  int* d_barrier = nullptr;
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
  std::vector<int64_t> stg_off_el;   // full-grad staging: param p at element offset (128-aligned)
  int64_t stg_elems = 0;
  int64_t push_bytes_bf16 = 0, push_bytes_fp8 = 0, pull_elems = 0;
  int64_t local_push_bf16 = 0, local_push_fp8 = 0;
  SymSlot* p2p_slot = nullptr;       // arena of the current P2P unshard
  SymSlot* gbuf = nullptr;           // zero-copy full-grad buffer (fsdp_full_grad_buffer)
  bool gbuf_sym = false;
  fsdp_dtype_t gbuf_dtype = FSDP_BFLOAT16;
  void* arena_base = nullptr;        // base of the unsharded tensors (either path)
};

namespace {

cudaEvent_t new_event(bool timing = false) {
  cudaEvent_t e;
  CUDA_CHECK(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  return e;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- profiling helpers
struct ProfScope {
  fsdp_mesh* m;
  int kind;
  cudaStream_t st;
  int64_t bytes;
  cudaEvent_t a = nullptr;
  ProfScope(fsdp_mesh* m_, int k, cudaStream_t s, int64_t b) : m(m_), kind(k), st(s), bytes(b) {
    if (!m->prof) return;
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

void prof_collect(fsdp_mesh* m) {
  for (auto& r : m->prof_recs) {
    CUDA_CHECK(cudaEventSynchronize(r.b));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
    m->prof_acc.launches[r.kind] += 1;
    m->prof_acc.total_ms[r.kind] += ms;
    m->prof_acc.bytes[r.kind] += r.bytes;
    m->ev_pool.push_back(r.a);
    m->ev_pool.push_back(r.b);
  }
  m->prof_recs.clear();
}

// ---- pools
Slot* acquire_slot(fsdp_mesh* m, std::vector<Slot*>& pool, size_t a_bytes, size_t b_bytes, int min_slots) {
  Slot* best = nullptr;
  int n_free = 0;
  for (Slot* s : pool) {
    if (s->in_use) continue;
    ++n_free;
    if (!best) { best = s; continue; }
    const bool s_done = !s->ever_used || cudaEventQuery(s->free_ev) == cudaSuccess;
    const bool b_done = !best->ever_used || cudaEventQuery(best->free_ev) == cudaSuccess;
    if (s_done != b_done) { if (s_done) best = s; continue; }
    if (s->last_use < best->last_use) best = s;
  }
  cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not sticky; clear it anyway
  const bool best_busy = best && best->ever_used && cudaEventQuery(best->free_ev) != cudaSuccess;
  cudaGetLastError();
  if (!best || ((int)pool.size() < min_slots && best_busy)) {
    Slot* s = new Slot();
    s->free_ev = new_event();
    pool.push_back(s);
    best = s;
  }
  if (best->a.cap < a_bytes || best->b.cap < b_bytes) {
    if (best->ever_used) CUDA_CHECK(cudaEventSynchronize(best->free_ev));   // growth: setup-time only
    best->a.ensure(a_bytes);
    best->b.ensure(b_bytes);
  }
  best->in_use = true;
  best->last_use = ++m->use_seq;
  return best;
}

void release_slot(Slot* s, cudaStream_t last_user) {
  CUDA_CHECK(cudaEventRecord(s->free_ev, last_user));
  s->ever_used = true;
  s->in_use = false;
}

void check_mesh(const fsdp_mesh* m) {
  if (!m) fail(FSDP_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (m->aborted) fail(FSDP_ERR_STATE, "mesh was aborted after a NCCL error/timeout");
}
void check_layer(const fsdp_layer* l) {
  if (!l) fail(FSDP_ERR_INVALID_ARGUMENT, "layer is NULL");
  check_mesh(l->mesh);
}
void check_param(const fsdp_layer* l, int p) {
  if (p < 0 || p >= l->P) fail(FSDP_ERR_INVALID_ARGUMENT, "param index out of range");
}

bool comm_ready(const fsdp_mesh* m) { return !m->local && m->W > 1; }

void ensure_registry(fsdp_mesh* m, int need) {
  if (need <= m->reg_cap) return;
  int cap = std::max(need, std::max(64, 2 * m->reg_cap));
  uint32_t* acc;
  float *amax, *scale;
  uint8_t* elig;
  CUDA_CHECK(cudaMalloc(&acc, sizeof(uint32_t) * cap));
  CUDA_CHECK(cudaMalloc(&amax, sizeof(float) * cap));
  CUDA_CHECK(cudaMalloc(&scale, sizeof(float) * cap));
  CUDA_CHECK(cudaMalloc(&elig, cap));
  CUDA_CHECK(cudaMemset(acc, 0, sizeof(uint32_t) * cap));
  CUDA_CHECK(cudaMemset(amax, 0, sizeof(float) * cap));
  CUDA_CHECK(cudaMemset(scale, 0, sizeof(float) * cap));
  CUDA_CHECK(cudaMemset(elig, 0, cap));
  if (m->reg_size) {
    CUDA_CHECK(cudaDeviceSynchronize());
    CUDA_CHECK(cudaMemcpy(acc, m->reg_acc, sizeof(uint32_t) * m->reg_size, cudaMemcpyDeviceToDevice));
    CUDA_CHECK(cudaMemcpy(amax, m->reg_amax, sizeof(float) * m->reg_size, cudaMemcpyDeviceToDevice));
    CUDA_CHECK(cudaMemcpy(scale, m->reg_scale, sizeof(float) * m->reg_size, cudaMemcpyDeviceToDevice));
    CUDA_CHECK(cudaMemcpy(elig, m->reg_elig, m->reg_size, cudaMemcpyDeviceToDevice));
  }
  // delayed-scaling state: amax history [cap][kHistMax], ring position, initialised flag
  float* hist;
  int32_t* pos;
  uint8_t* hinit;
  CUDA_CHECK(cudaMalloc(&hist, sizeof(float) * (size_t)cap * kHistMax));
  CUDA_CHECK(cudaMalloc(&pos, sizeof(int32_t) * cap));
  CUDA_CHECK(cudaMalloc(&hinit, cap));
  CUDA_CHECK(cudaMemset(hist, 0, sizeof(float) * (size_t)cap * kHistMax));
  CUDA_CHECK(cudaMemset(pos, 0, sizeof(int32_t) * cap));
  CUDA_CHECK(cudaMemset(hinit, 0, cap));
  if (m->reg_size) {
    CUDA_CHECK(cudaMemcpy(hist, m->reg_hist, sizeof(float) * (size_t)m->reg_size * kHistMax, cudaMemcpyDeviceToDevice));
    CUDA_CHECK(cudaMemcpy(pos, m->reg_pos, sizeof(int32_t) * m->reg_size, cudaMemcpyDeviceToDevice));
    CUDA_CHECK(cudaMemcpy(hinit, m->reg_hinit, m->reg_size, cudaMemcpyDeviceToDevice));
  }
  cudaFree(m->reg_acc); cudaFree(m->reg_amax); cudaFree(m->reg_scale); cudaFree(m->reg_elig);
  cudaFree(m->reg_hist); cudaFree(m->reg_pos); cudaFree(m->reg_hinit);
  m->reg_acc = acc; m->reg_amax = amax; m->reg_scale = scale; m->reg_elig = elig;
  m->reg_hist = hist; m->reg_pos = pos; m->reg_hinit = hinit;
  m->reg_cap = cap;
  for (auto* ps : m->presets) { ps->tiles.release(); cudaFree(ps->idx); delete ps; }
  m->presets.clear();
}

void clear_presets(fsdp_mesh* m) {
  for (auto* ps : m->presets) { ps->tiles.release(); cudaFree(ps->idx); delete ps; }
  m->presets.clear();
}

int64_t dtype_size(fsdp_dtype_t d) { return d == FSDP_FLOAT32 ? 4 : (d == FSDP_BFLOAT16 ? 2 : 1); }

// ---- symmetric memory over CUDA IPC (collective helpers; every rank calls them in the
// same order, which the deterministic FSDP call sequence guarantees)
void mesh_barrier(fsdp_mesh* m) {
  NCCL_CHECK(ncclAllReduce(m->d_barrier, m->d_barrier, 1, ncclInt32, ncclSum, m->comm_ag, m->s_ag));
  CUDA_CHECK(cudaStreamSynchronize(m->s_ag));
}

// all ranks agree that `ok` holds everywhere
bool mesh_all_ok(fsdp_mesh* m, bool ok) {
  int v = ok ? 1 : 0;
  CUDA_CHECK(cudaMemcpy(m->d_barrier, &v, sizeof(int), cudaMemcpyHostToDevice));
  NCCL_CHECK(ncclAllReduce(m->d_barrier, m->d_barrier, 1, ncclInt32, ncclMin, m->comm_ag, m->s_ag));
  CUDA_CHECK(cudaStreamSynchronize(m->s_ag));
  CUDA_CHECK(cudaMemcpy(&v, m->d_barrier, sizeof(int), cudaMemcpyDeviceToHost));
  return v == 1;
}

// Rank-local (aborted mesh): unmap the peers' copies and free the local one, no barrier.
void sym_free_local(fsdp_mesh* m, SymBuf& b) {
  for (int r = 0; r < m->W; ++r)
    if (r != m->rank && r < (int)b.peers.size() && b.peers[r]) cudaIpcCloseMemHandle(b.peers[r]);
  if (b.local) cudaFree(b.local);
  cudaGetLastError();
  b = SymBuf();
}

// Collective: unmap the peers' copies, wait until every rank did, then free the local one.
void sym_free(fsdp_mesh* m, SymBuf& b) {
  for (int r = 0; r < m->W; ++r)
    if (r != m->rank && r < (int)b.peers.size() && b.peers[r]) cudaIpcCloseMemHandle(b.peers[r]);
  cudaGetLastError();
  mesh_barrier(m);
  if (b.local) cudaFree(b.local);
  b = SymBuf();
}

// Returns false (on every rank) if any rank failed to allocate or map.
bool sym_alloc(fsdp_mesh* m, SymBuf& b, size_t bytes) {
  bool ok = cudaMalloc(&b.local, bytes + 256) == cudaSuccess;
  cudaIpcMemHandle_t h{};
  if (ok) ok = cudaMemset(b.local, 0, bytes + 256) == cudaSuccess;
  if (ok) ok = cudaIpcGetMemHandle(&h, b.local) == cudaSuccess;
  cudaGetLastError();
  uint8_t* d = nullptr;
  CUDA_CHECK(cudaMalloc(&d, sizeof(h) * m->W));
  CUDA_CHECK(cudaMemcpy(d + sizeof(h) * m->rank, &h, sizeof(h), cudaMemcpyHostToDevice));
  NCCL_CHECK(ncclAllGather(d + sizeof(h) * m->rank, d, sizeof(h), ncclUint8, m->comm_ag, m->s_ag));
  CUDA_CHECK(cudaStreamSynchronize(m->s_ag));
  std::vector<cudaIpcMemHandle_t> hs(m->W);
  CUDA_CHECK(cudaMemcpy(hs.data(), d, sizeof(h) * m->W, cudaMemcpyDeviceToHost));
  cudaFree(d);
  b.peers.assign(m->W, nullptr);
  b.bytes = bytes;
  if (ok) {
    b.peers[m->rank] = b.local;
    for (int r = 0; r < m->W && ok; ++r) {
      if (r == m->rank) continue;
      void* p = nullptr;
      ok = cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      cudaGetLastError();
      b.peers[r] = ok ? p : nullptr;
    }
  }
  if (!mesh_all_ok(m, ok)) {
    sym_free(m, b);
    return false;
  }
  return true;
}

fsdpp::FlagPtrs flag_remote(fsdp_mesh* m, int kind, int slot) {
  fsdpp::FlagPtrs f{};
  const size_t off = ((size_t)kind * kFlagSlots + slot) * fsdpp::kMaxRanks;
  for (int r = 0; r < m->W; ++r) f.p[r] = (unsigned long long*)m->flags.peers[r] + off;
  return f;
}
unsigned long long* flag_local(fsdp_mesh* m, int kind, int slot) {
  return (unsigned long long*)m->flags.local + ((size_t)kind * kFlagSlots + slot) * fsdpp::kMaxRanks;
}

// Deterministic choice: the lowest-index free slot (same on every rank, since in_use
// depends only on the call sequence); grows / creates slots collectively.
SymSlot* acquire_sym_slot(fsdp_mesh* m, std::vector<SymSlot*>& pool, size_t bytes, int prefer = -1) {
  SymSlot* s = nullptr;
  while (prefer >= (int)pool.size() && (int)pool.size() < kPoolSlots) {
    SymSlot* n = new SymSlot();
    n->free_ev = new_event();
    n->index = (int)pool.size();
    pool.push_back(n);
  }
  if (prefer >= 0 && prefer < (int)pool.size() && !pool[prefer]->in_use) s = pool[prefer];
  for (size_t i = 0; !s && i < pool.size(); ++i)
    if (!pool[i]->in_use) s = pool[i];
  if (!s) {
    if ((int)pool.size() >= kPoolSlots) fail(FSDP_ERR_STATE, "too many unsharded layers / pending reduce-scatters at once");
    s = new SymSlot();
    s->free_ev = new_event();
    s->index = (int)pool.size();
    pool.push_back(s);
  }
  if (s->buf.bytes < bytes) {   // collective (re)allocation; setup-time only
    if (s->ever_used) CUDA_CHECK(cudaEventSynchronize(s->free_ev));
    CUDA_CHECK(cudaDeviceSynchronize());
    mesh_barrier(m);
    if (s->buf.local || !s->buf.peers.empty()) sym_free(m, s->buf);
    if (!sym_alloc(m, s->buf, bytes)) fail(FSDP_ERR_OUT_OF_MEMORY, "symmetric buffer allocation/mapping failed");
  }
  s->in_use = true;
  return s;
}

fsdpp::PeerPtrs peer_ptrs(const fsdp_mesh* m, const SymBuf& b) {
  fsdpp::PeerPtrs p{};
  for (int r = 0; r < m->W; ++r) p.p[r] = (uint8_t*)b.peers[r];
  return p;
}

void p2p_teardown(fsdp_mesh* m) {
  if (!m->p2p_ok) return;
  CUDA_CHECK(cudaDeviceSynchronize());
  mesh_barrier(m);   // every rank's kernels are done with every peer buffer
  for (auto* pool : {&m->p2p_ag, &m->p2p_rs}) {
    for (SymSlot* s : *pool) {
      if (s->buf.local || !s->buf.peers.empty()) sym_free(m, s->buf);
      if (s->free_ev) cudaEventDestroy(s->free_ev);
      delete s;
    }
    pool->clear();
  }
  sym_free(m, m->flags);
  m->p2p_ok = false;
}

// ---- K4 / K5 launches (fsdp_shard enforces P <= kMaxPtrs, one pointer array per launch)
void launch_copy_out_all(fsdp_layer* l, bool fp8, const void* ag, void* const* outs, cudaStream_t st) {
  const DevTiles& T = fp8 ? l->t_cout_fp8 : l->t_cout_bf16;
  fsdpk::PtrArray pa{};
  for (int p = 0; p < l->P; ++p) pa.p[p] = outs[p];
  CUDA_CHECK(fsdpk::launch_copy_out(T.d, T.n, ag, pa, l->mesh->cfg, st));
}

void launch_rs_copy_in_all(fsdp_layer* l, const void* const* grads, bool grad_bf16, void* rs_in, bool out_bf16,
                           bool mean, cudaStream_t st) {
  fsdpk::PtrArray pa{};
  for (int p = 0; p < l->P; ++p) pa.p[p] = grads[p];
  CUDA_CHECK(fsdpk::launch_rs_copy_in(l->t_rsin.d, l->t_rsin.n, pa, grad_bf16, rs_in, out_bf16, mean,
                                      l->mesh->W * l->mesh->R,
                                      l->mesh->cfg, st));
}

int64_t cin_bytes(const fsdp_layer* l, bool fp8) { return fp8 ? l->bytes_cin_fp8 : 6 * l->L.S; }
int64_t slot_bytes(const fsdp_layer* l, bool fp8) { return fp8 ? l->L.S_bytes_fp8 : 2 * l->L.S; }

void do_copy_in(fsdp_layer* l, bool fp8, const float* scales, void* dst, cudaStream_t st) {
  fsdp_mesh* m = l->mesh;
  ProfScope ps(m, FSDP_PROF_COPY_IN, st, cin_bytes(l, fp8));
  if (fp8) CUDA_CHECK(fsdpk::launch_copy_in_fp8(l->t_cin_fp8.d, l->t_cin_fp8.n, l->shard, dst, scales, m->cfg, st));
  else CUDA_CHECK(fsdpk::launch_copy_in_bf16(l->shard, dst, l->L.S, m->cfg, st));
  ps.done();
}

void validate_grads(const fsdp_layer* l, const void* const* grads, fsdp_dtype_t gd, fsdp_dtype_t rd) {
  if (!grads) fail(FSDP_ERR_INVALID_ARGUMENT, "full_grads is NULL");
  for (int p = 0; p < l->P; ++p)
    if (!grads[p] && l->L.numel[p] > 0) fail(FSDP_ERR_INVALID_ARGUMENT, "full_grads[p] is NULL");
  if (gd != FSDP_BFLOAT16 && gd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "grad_dtype must be BFLOAT16 or FLOAT32");
  if (rd != FSDP_BFLOAT16 && rd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "reduce_dtype must be FLOAT32 or BFLOAT16");
}

}  // namespace

extern "C" {

int32_t fsdp_abi_version(void) { return FSDP_B200_ABI_VERSION; }
const char* fsdp_last_error(void) { return g_last_error.c_str(); }

const char* fsdp_status_string(fsdp_status_t s) {
  switch (s) {
    case FSDP_OK: return "FSDP_OK";
    case FSDP_ERR_INVALID_ARGUMENT: return "FSDP_ERR_INVALID_ARGUMENT";
    case FSDP_ERR_SHAPE: return "FSDP_ERR_SHAPE";
    case FSDP_ERR_DTYPE: return "FSDP_ERR_DTYPE";
    case FSDP_ERR_STATE: return "FSDP_ERR_STATE";
    case FSDP_ERR_OUT_OF_MEMORY: return "FSDP_ERR_OUT_OF_MEMORY";
    case FSDP_ERR_CUDA: return "FSDP_ERR_CUDA";
    case FSDP_ERR_NCCL: return "FSDP_ERR_NCCL";
    case FSDP_ERR_TIMEOUT: return "FSDP_ERR_TIMEOUT";
    case FSDP_ERR_NONFINITE: return "FSDP_ERR_NONFINITE";
    case FSDP_ERR_UNAVAILABLE: return "FSDP_ERR_UNAVAILABLE";
  }
  return "FSDP_ERR_UNKNOWN";
}

fsdp_status_t fsdp_layout_compute(int32_t n_params, const fsdp_param_desc_t* descs, int32_t world_size,
                                  int32_t rank, fsdp_param_meta_t* out_metas, int64_t* out_S,
                                  int64_t* out_S_bytes_fp8, uint64_t* out_hash) {
  return guarded([&] {
    Layout L;
    const char* msg = "";
    fsdp_status_t st = fsdpl::compute_layout(n_params, descs, world_size, rank, &L, &msg);
    if (st != FSDP_OK) fail(st, msg);
    if (out_metas) std::copy(L.metas.begin(), L.metas.end(), out_metas);
    if (out_S) *out_S = L.S;
    if (out_S_bytes_fp8) *out_S_bytes_fp8 = L.S_bytes_fp8;
    if (out_hash) *out_hash = L.hash;
  });
}

fsdp_status_t fsdp_get_unique_id(uint8_t id[FSDP_UNIQUE_ID_BYTES]) {
  return guarded([&] {
    if (!id) fail(FSDP_ERR_INVALID_ARGUMENT, "id is NULL");
    static_assert(sizeof(ncclUniqueId) == FSDP_UNIQUE_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    NCCL_CHECK(ncclGetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
  });
}

static void mesh_common_init(fsdp_mesh* m) {
  int prio_lo = 0, prio_hi = 0;
  CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  for (cudaStream_t* s : {&m->s_cin, &m->s_ag, &m->s_cout, &m->s_rsc, &m->s_rs})
    CUDA_CHECK(cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, prio_hi));
  int sms = 0;
  CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device));
  // persistent grids: CTAs per SM (256 threads each); FSDP_B200_CTAS_PER_SM tunes it
  int per_sm = 0;   // 0: each kernel's tuned value (kernels.h)
  if (const char* e = std::getenv("FSDP_B200_CTAS_PER_SM")) per_sm = std::max(1, std::min(16, std::atoi(e)));
  m->cfg.sms = sms;
  m->cfg.per_sm = per_sm;
  // default: TMA bulk push (4), bulk RS copy-in (8) and, for zero-copy reduce-scatters, bulk
  // pull (2) — measured best (profiles/r06, r07); FSDP_B200_VARIANT overrides (0 = plain ld/st)
  m->cfg.variant = 14;
  if (const char* e = std::getenv("FSDP_B200_VARIANT")) m->cfg.variant = std::atoi(e);
  m->cfg.grid_cap = sms * (per_sm > 0 ? per_sm : 4);
  CUDA_CHECK(cudaMalloc(&m->d_err, sizeof(int)));
  CUDA_CHECK(cudaMemset(m->d_err, 0, sizeof(int)));
  m->ev_pre_call = new_event();
  m->ev_pre_done = new_event();
  CUDA_CHECK(cudaMalloc(&m->d_barrier, sizeof(int)));
  CUDA_CHECK(cudaMemset(m->d_barrier, 0, sizeof(int)));
}

// P2P capability: W in [2, 8] and every rank can map every peer's buffer (collective).
static void p2p_init(fsdp_mesh* m) {
  if (m->local || m->W < 2 || m->W > 8) return;
  const size_t fbytes = sizeof(unsigned long long) * FK_NUM * kFlagSlots * fsdpp::kMaxRanks;
  m->p2p_ok = sym_alloc(m, m->flags, fbytes);
  const char* env = std::getenv("FSDP_B200_ALGO");
  const bool want_nccl = env && std::string(env) == "nccl";
  m->algo = (m->p2p_ok && !want_nccl) ? FSDP_ALGO_P2P : FSDP_ALGO_NCCL;
  if (const char* t = std::getenv("FSDP_B200_P2P_TIMEOUT_MS"))
    m->p2p_timeout_ns = (unsigned long long)std::max(1L, std::atol(t)) * 1000000ull;
}

static fsdp_status_t mesh_init_impl(const uint8_t* id, int32_t W, int32_t rank, int32_t dev, bool local,
                                    fsdp_mesh_t** out, int32_t shard_size = 0) {
  return guarded([&] {
    if (!out) fail(FSDP_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (W < 1 || rank < 0 || rank >= W) fail(FSDP_ERR_INVALID_ARGUMENT, "invalid world_size/rank");
    if (!local && !id) fail(FSDP_ERR_INVALID_ARGUMENT, "unique id is NULL");
    if (shard_size <= 0) shard_size = W;
    if (W % shard_size != 0) fail(FSDP_ERR_INVALID_ARGUMENT, "shard_size must divide world_size");
    int ndev = 0;
    CUDA_CHECK(cudaGetDeviceCount(&ndev));
    if (dev < 0 || dev >= ndev) fail(FSDP_ERR_INVALID_ARGUMENT, "cuda_device out of range");
    DeviceGuard g(dev);
    auto* m = new fsdp_mesh();
    m->W = shard_size;              // the Shard(0) degree
    m->rank = rank % shard_size;    // shard rank (replica dimension outer, R15)
    m->R = W / shard_size;
    m->rep = rank / shard_size;
    m->device = dev;
    m->local = local;
    try {
      mesh_common_init(m);
      if (!local) {
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        if (m->R == 1) {
          NCCL_CHECK(ncclCommInitRank(&m->comm_ag, W, u, rank));
        } else {   // HSDP: world comm -> shard group (color = replica) and replica group (color = shard rank)
          NCCL_CHECK(ncclCommInitRank(&m->comm_world, W, u, rank));
          NCCL_CHECK(ncclCommSplit(m->comm_world, m->rep, m->rank, &m->comm_ag, nullptr));
          NCCL_CHECK(ncclCommSplit(m->comm_world, m->rank, m->rep, &m->comm_rep, nullptr));
        }
        NCCL_CHECK(ncclCommSplit(m->comm_ag, 0, m->rank, &m->comm_rs, nullptr));
        p2p_init(m);
      }
    } catch (...) {
      fsdp_mesh_destroy(m);
      throw;
    }
    *out = m;
  });
}

fsdp_status_t fsdp_mesh_init(const uint8_t id[FSDP_UNIQUE_ID_BYTES], int32_t world_size, int32_t rank,
                             int32_t cuda_device, fsdp_mesh_t** out) {
  return mesh_init_impl(id, world_size, rank, cuda_device, false, out);
}

fsdp_status_t fsdp_mesh_init_local(int32_t world_size, int32_t rank, int32_t cuda_device, fsdp_mesh_t** out) {
  return mesh_init_impl(nullptr, world_size, rank, cuda_device, true, out);
}

fsdp_status_t fsdp_mesh_init_hsdp(const uint8_t id[FSDP_UNIQUE_ID_BYTES], int32_t world_size, int32_t rank,
                                  int32_t shard_size, int32_t cuda_device, fsdp_mesh_t** out) {
  if (shard_size < 1) {
    g_last_error = "shard_size must be >= 1";
    return FSDP_ERR_INVALID_ARGUMENT;
  }
  return mesh_init_impl(id, world_size, rank, cuda_device, false, out, shard_size);
}

fsdp_status_t fsdp_mesh_info_hsdp(const fsdp_mesh_t* m, int32_t* R, int32_t* rep) {
  return guarded([&] {
    if (!m) fail(FSDP_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (R) *R = m->R;
    if (rep) *rep = m->rep;
  });
}

fsdp_status_t fsdp_mesh_destroy(fsdp_mesh_t* m) {
  return guarded([&] {
    if (!m) return;
    if (!m->layers.empty()) fail(FSDP_ERR_STATE, "destroy all layers of the mesh first");
    DeviceGuard g(m->device);
    for (cudaStream_t s : {m->s_cin, m->s_ag, m->s_cout, m->s_rsc, m->s_rs})
      if (s) cudaStreamSynchronize(s);
    if (!m->aborted) {
      p2p_teardown(m);
    } else {   // rank-local release, no collective step
      for (auto* pool : {&m->p2p_ag, &m->p2p_rs}) {
        for (SymSlot* s : *pool) {
          sym_free_local(m, s->buf);
          if (s->free_ev) cudaEventDestroy(s->free_ev);
          delete s;
        }
        pool->clear();
      }
      sym_free_local(m, m->flags);
    }
    for (auto* pool : {&m->ag_slots, &m->rs_slots})
      for (Slot* s : *pool) { s->a.release(); s->b.release(); if (s->free_ev) cudaEventDestroy(s->free_ev); delete s; }
    clear_presets(m);
    for (auto& r : m->prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : m->ev_pool) cudaEventDestroy(e);
    cudaFree(m->reg_acc); cudaFree(m->reg_amax); cudaFree(m->reg_scale); cudaFree(m->reg_elig);
    cudaFree(m->reg_hist); cudaFree(m->reg_pos); cudaFree(m->reg_hinit);
    cudaFree(m->d_err);
    cudaFree(m->d_barrier);
    if (m->ev_pre_call) cudaEventDestroy(m->ev_pre_call);
    if (m->ev_pre_done) cudaEventDestroy(m->ev_pre_done);
    if (m->comm_rs) { if (m->aborted) ncclCommAbort(m->comm_rs); else ncclCommDestroy(m->comm_rs); }
    if (m->comm_ag) { if (m->aborted) ncclCommAbort(m->comm_ag); else ncclCommDestroy(m->comm_ag); }
    for (ncclComm_t c : {m->comm_rep, m->comm_world})
      if (c) { if (m->aborted) ncclCommAbort(c); else ncclCommDestroy(c); }
    for (cudaStream_t s : {m->s_cin, m->s_ag, m->s_cout, m->s_rsc, m->s_rs})
      if (s) cudaStreamDestroy(s);
    delete m;
  });
}

fsdp_status_t fsdp_mesh_info(const fsdp_mesh_t* m, int32_t* W, int32_t* rank, int32_t* dev) {
  return guarded([&] {
    if (!m) fail(FSDP_ERR_INVALID_ARGUMENT, "mesh is NULL");
    if (W) *W = m->W;
    if (rank) *rank = m->rank;
    if (dev) *dev = m->device;
  });
}

fsdp_status_t fsdp_mesh_abort(fsdp_mesh_t* m) {
  return guarded([&] {
    if (!m) fail(FSDP_ERR_INVALID_ARGUMENT, "mesh is NULL");
    m->aborted = true;
    for (ncclComm_t* c : {&m->comm_ag, &m->comm_rs, &m->comm_rep, &m->comm_world})
      if (*c) {
        ncclCommAbort(*c);
        *c = nullptr;
      }
  });
}

fsdp_status_t fsdp_mesh_set_algo(fsdp_mesh_t* m, int32_t algo) {
  return guarded([&] {
    check_mesh(m);
    if (algo != FSDP_ALGO_NCCL && algo != FSDP_ALGO_P2P) fail(FSDP_ERR_INVALID_ARGUMENT, "unknown algo");
    for (auto* l : m->layers)
      if (l->state != SHARDED || l->rs_pending) fail(FSDP_ERR_STATE, "a layer is unsharded or has a pending reduce-scatter");
    if (algo == FSDP_ALGO_P2P && !m->p2p_ok) fail(FSDP_ERR_UNAVAILABLE, "P2P needs 2 <= W <= 8 ranks whose GPUs can map each other's memory");
    m->algo = algo;
  });
}

fsdp_status_t fsdp_mesh_get_algo(const fsdp_mesh_t* m, int32_t* algo) {
  return guarded([&] {
    if (!m || !algo) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    *algo = m->algo;
  });
}

fsdp_status_t fsdp_mesh_synchronize(fsdp_mesh_t* m, int64_t timeout_ms) {
  return guarded([&] {
    check_mesh(m);
    DeviceGuard g(m->device);
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t ss[] = {m->s_cin, m->s_ag, m->s_cout, m->s_rsc, m->s_rs};
    for (;;) {
      bool idle = true;
      for (cudaStream_t s : ss) {
        cudaError_t e = cudaStreamQuery(s);
        if (e == cudaErrorNotReady) { idle = false; continue; }
        if (e != cudaSuccess) fail(FSDP_ERR_CUDA, std::string("stream error: ") + cudaGetErrorString(e));
      }
      if (comm_ready(m)) {
        for (ncclComm_t c : {m->comm_ag, m->comm_rs}) {
          ncclResult_t ar = ncclSuccess;
          NCCL_CHECK(ncclCommGetAsyncError(c, &ar));
          if (ar != ncclSuccess) {
            m->aborted = true;
            fail(FSDP_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(ar));
          }
        }
      }
      if (idle) break;
      if (timeout_ms > 0 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms)) {
        m->aborted = true;
        if (m->comm_ag) ncclCommAbort(m->comm_ag);
        if (m->comm_rs) ncclCommAbort(m->comm_rs);
        m->comm_ag = m->comm_rs = nullptr;
        fail(FSDP_ERR_TIMEOUT, "mesh streams did not drain before the timeout; communicators aborted");
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    int err = 0;
    CUDA_CHECK(cudaMemcpy(&err, m->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
      CUDA_CHECK(cudaMemset(m->d_err, 0, sizeof(int)));
      if ((err & 0xFF) == 2) {   // a P2P handshake gave up waiting for a peer
        m->aborted = true;
        fail(FSDP_ERR_TIMEOUT, "P2P handshake timed out waiting for shard rank " + std::to_string(err >> 8) +
                                   " (a rank skipped or diverged from the collective call sequence); mesh aborted");
      }
      fail(FSDP_ERR_NONFINITE, "non-finite fp8 amax seen by fsdp_precompute_fp8_scales (SPEC.md:38)");
    }
  });
}

fsdp_status_t fsdp_profile_enable(fsdp_mesh_t* m, int32_t on) {
  return guarded([&] {
    check_mesh(m);
    m->prof = on != 0;
  });
}

fsdp_status_t fsdp_profile_read(fsdp_mesh_t* m, fsdp_profile_t* out, int32_t reset) {
  return guarded([&] {
    check_mesh(m);
    DeviceGuard g(m->device);
    prof_collect(m);
    if (out) *out = m->prof_acc;
    if (reset) m->prof_acc = fsdp_profile_t{};
  });
}

// ------------------------------------------------------------------------- shard
fsdp_status_t fsdp_shard(fsdp_mesh_t* m, int32_t n, const fsdp_param_desc_t* descs,
                         const float* const* full_params, fsdp_layer_t** out) {
  return guarded([&] {
    check_mesh(m);
    if (!out) fail(FSDP_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (n < 1) fail(FSDP_ERR_INVALID_ARGUMENT, "a unit needs at least one parameter");
    Layout L;
    const char* msg = "";
    fsdp_status_t st = fsdpl::compute_layout(n, descs, m->W, m->rank, &L, &msg);
    if (st != FSDP_OK) fail(st, msg);
    if (n > fsdpk::kMaxPtrs) fail(FSDP_ERR_UNAVAILABLE, "units with more than 512 parameters are not supported in this build");
    DeviceGuard g(m->device);
    if (comm_ready(m)) {  // all ranks must agree on the unit ("shape mismatch across members")
      uint64_t* d = nullptr;
      CUDA_CHECK(cudaMalloc(&d, sizeof(uint64_t) * m->W));
      CUDA_CHECK(cudaMemcpy(d + m->rank, &L.hash, sizeof(uint64_t), cudaMemcpyHostToDevice));
      NCCL_CHECK(ncclAllGather(d + m->rank, d, 8, ncclUint8, m->comm_ag, m->s_ag));
      std::vector<uint64_t> h(m->W);
      CUDA_CHECK(cudaStreamSynchronize(m->s_ag));
      CUDA_CHECK(cudaMemcpy(h.data(), d, sizeof(uint64_t) * m->W, cudaMemcpyDeviceToHost));
      cudaFree(d);
      for (uint64_t x : h)
        if (x != L.hash) fail(FSDP_ERR_SHAPE, "ranks disagree on the unit's parameter shapes (layout hash mismatch)");
    }
    auto* l = new fsdp_layer();
    l->mesh = m;
    l->P = n;
    l->descs.assign(descs, descs + n);
    l->L = std::move(L);
    try {
      const Layout& Ly = l->L;
      const size_t sbytes = sizeof(float) * (size_t)std::max<int64_t>(Ly.S, 16);
      CUDA_CHECK(cudaMalloc(&l->shard, sbytes));
      CUDA_CHECK(cudaMalloc(&l->grad, sbytes));
      CUDA_CHECK(cudaMemset(l->shard, 0, sbytes));
      CUDA_CHECK(cudaMemset(l->grad, 0, sbytes));
      if (full_params) {
        for (int p = 0; p < n; ++p) {
          const auto& mt = Ly.metas[p];
          const int64_t cnt = mt.row_count * mt.rest;
          if (!full_params[p] || cnt == 0) continue;
          CUDA_CHECK(cudaMemcpy(l->shard + mt.elem_offset, full_params[p] + mt.row_begin * mt.rest,
                                sizeof(float) * cnt, cudaMemcpyDefault));
        }
      }
      l->t_cin_fp8.upload(fsdpl::tiles_copy_in_fp8(Ly));
      l->t_cout_bf16.upload(fsdpl::tiles_copy_out(Ly, false, &l->t_cout_bf16.first));
      l->t_cout_fp8.upload(fsdpl::tiles_copy_out(Ly, true, &l->t_cout_fp8.first));
      l->t_rsin.upload(fsdpl::tiles_rs_copy_in(Ly, &l->t_rsin.first));
      l->stg_off_el = fsdpl::staging_offsets(Ly, &l->stg_elems);
      l->t_push_bf16.upload(fsdpl::tiles_push(Ly, false));
      l->t_push_fp8.upload(fsdpl::tiles_push(Ly, true));
      l->t_pull.upload(fsdpl::tiles_pull(Ly, l->stg_off_el));
      l->t_stage_bf16.upload(fsdpl::tiles_stage(Ly, l->stg_off_el, 2));
      l->t_stage_fp32.upload(fsdpl::tiles_stage(Ly, l->stg_off_el, 4));
      for (int p = 0; p < n; ++p) {
        const int64_t cnt = Ly.metas[p].row_count * Ly.metas[p].rest;
        const int64_t es8 = Ly.fp8[p] ? 1 : 2;
        l->push_bytes_bf16 += (int64_t)(m->W - 1) * cnt * 2;      // NVLink egress
        l->push_bytes_fp8 += (int64_t)(m->W - 1) * cnt * es8;
        l->local_push_bf16 += cnt * (4 + 2);                        // W=1: HBM read + write
        l->local_push_fp8 += cnt * (4 + es8);
        l->pull_elems += cnt;
      }
      for (int p = 0; p < n; ++p) {
        const int64_t es = Ly.fp8[p] ? 1 : 2;
        l->bytes_cin_fp8 += Ly.metas[p].padded_numel * (4 + es);
        l->bytes_cout_bf16 += 2 * 2 * Ly.numel[p];
        l->bytes_cout_fp8 += 2 * es * Ly.numel[p];
        l->grad_numel_total += Ly.numel[p];
      }
      // fp8 registry entries [reg_base, reg_base + P)
      ensure_registry(m, m->reg_size + n);
      l->reg_base = m->reg_size;
      m->reg_size += n;
      CUDA_CHECK(cudaMemcpy(m->reg_elig + l->reg_base, Ly.fp8.data(), n, cudaMemcpyHostToDevice));
      std::vector<int32_t> idx(n);
      for (int p = 0; p < n; ++p) idx[p] = p;
      CUDA_CHECK(cudaMalloc(&l->d_idx_local, sizeof(int32_t) * n));
      CUDA_CHECK(cudaMemcpy(l->d_idx_local, idx.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
      for (cudaEvent_t* e : {&l->ev_call, &l->ev_cin, &l->ev_ag, &l->ev_done, &l->ev_rcall, &l->ev_k5, &l->ev_rs_done})
        *e = new_event();
      CUDA_CHECK(cudaDeviceSynchronize());
    } catch (...) {
      m->layers.push_back(l);
      fsdp_layer_destroy(l);
      throw;
    }
    m->layers.push_back(l);
    *out = l;
  });
}

fsdp_status_t fsdp_layer_destroy(fsdp_layer_t* l) {
  return guarded([&] {
    if (!l) return;
    fsdp_mesh* m = l->mesh;
    if (l->state != SHARDED) fail(FSDP_ERR_STATE, "reshard the layer before destroying it");
    DeviceGuard g(m->device);
    for (cudaStream_t s : {m->s_cin, m->s_ag, m->s_cout, m->s_rsc, m->s_rs}) cudaStreamSynchronize(s);
    cudaFree(l->shard);
    cudaFree(l->grad);
    cudaFree(l->d_idx_local);
    l->t_cin_fp8.release(); l->t_cout_bf16.release(); l->t_cout_fp8.release(); l->t_rsin.release();
    l->t_push_bf16.release(); l->t_push_fp8.release(); l->t_pull.release(); l->t_stage_bf16.release();
    l->t_stage_fp32.release();
    if (l->gbuf) {
      if (l->gbuf_sym && !m->aborted) sym_free(m, l->gbuf->buf);   // collective
      else if (l->gbuf_sym) sym_free_local(m, l->gbuf->buf);
      else cudaFree(l->gbuf->buf.local);
      if (l->gbuf->free_ev) cudaEventDestroy(l->gbuf->free_ev);
      delete l->gbuf;
      l->gbuf = nullptr;
    }
    for (cudaEvent_t e : {l->ev_call, l->ev_cin, l->ev_ag, l->ev_done, l->ev_rcall, l->ev_k5, l->ev_rs_done})
      if (e) cudaEventDestroy(e);
    m->layers.erase(std::remove(m->layers.begin(), m->layers.end(), l), m->layers.end());
    clear_presets(m);
    delete l;
  });
}

fsdp_status_t fsdp_layer_info(const fsdp_layer_t* l, int32_t* n, int64_t* S, int64_t* Sb) {
  return guarded([&] {
    if (!l) fail(FSDP_ERR_INVALID_ARGUMENT, "layer is NULL");
    if (n) *n = l->P;
    if (S) *S = l->L.S;
    if (Sb) *Sb = l->L.S_bytes_fp8;
  });
}

fsdp_status_t fsdp_param_meta(const fsdp_layer_t* l, int32_t p, fsdp_param_meta_t* out) {
  return guarded([&] {
    if (!l) fail(FSDP_ERR_INVALID_ARGUMENT, "layer is NULL");
    check_param(l, p);
    if (!out) fail(FSDP_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = l->L.metas[p];
  });
}

fsdp_status_t fsdp_sharded_param(const fsdp_layer_t* l, int32_t p, float** dev) {
  return guarded([&] {
    if (!l || !dev) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    check_param(l, p);
    *dev = l->shard + l->L.metas[p].elem_offset;
  });
}

fsdp_status_t fsdp_sharded_flat(const fsdp_layer_t* l, float** dev) {
  return guarded([&] {
    if (!l || !dev) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    *dev = l->shard;
  });
}

// ------------------------------------------------------------------------- fp8 scales
// history_len == 0: dynamic scaling; > 0: delayed scaling with that amax history length.
static fsdp_status_t precompute_impl(fsdp_mesh_t* m, fsdp_layer_t* const* layers, int32_t n, void* stream,
                                     int32_t history_len) {
  return guarded([&] {
    check_mesh(m);
    if (history_len < 0 || history_len > kHistMax) fail(FSDP_ERR_INVALID_ARGUMENT, "history_len must be in [1, 64]");
    if (history_len > 0 && m->hist_len > 0 && history_len != m->hist_len)
      fail(FSDP_ERR_INVALID_ARGUMENT, "the amax history length is fixed at the first delayed precompute");
    if (n < 0 || (n > 0 && !layers)) fail(FSDP_ERR_INVALID_ARGUMENT, "layers is NULL");
    for (int i = 0; i < n; ++i) {
      if (!layers[i] || layers[i]->mesh != m) fail(FSDP_ERR_INVALID_ARGUMENT, "layer does not belong to this mesh");
    }
    if (m->local && m->W > 1) fail(FSDP_ERR_UNAVAILABLE, "local mesh with world_size > 1 has no communicator");
    DeviceGuard g(m->device);
    std::vector<fsdp_layer*> key(layers, layers + n);
    fsdp_mesh::PreSet* ps = nullptr;
    for (auto* c : m->presets) if (c->layers == key) { ps = c; break; }
    if (!ps) {
      ps = new fsdp_mesh::PreSet();
      ps->layers = key;
      std::vector<Tile> tiles;
      std::vector<int32_t> idx;
      for (fsdp_layer* l : key) {
        fsdpl::append_tiles_amax(l->L, l->shard, l->reg_base, &tiles);
        for (int p = 0; p < l->P; ++p) {
          idx.push_back(l->reg_base + p);
          if (l->L.fp8[p]) ps->bytes += 4 * l->L.metas[p].padded_numel;
        }
      }
      ps->tiles.upload(tiles);
      ps->nidx = (int)idx.size();
      if (ps->nidx) {
        CUDA_CHECK(cudaMalloc(&ps->idx, sizeof(int32_t) * idx.size()));
        CUDA_CHECK(cudaMemcpy(ps->idx, idx.data(), sizeof(int32_t) * idx.size(), cudaMemcpyHostToDevice));
      }
      m->presets.push_back(ps);
    }
    // precompute runs on s_rs (the stream owning comm_rs), ordered after `stream`, and
    // `stream` waits for it: K1 over all layers -> all-reduce(max) -> K1b
    cudaStream_t st = as_stream(stream);
    CUDA_CHECK(cudaEventRecord(m->ev_pre_call, st));
    CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, m->ev_pre_call, 0));
    {
      ProfScope pa(m, FSDP_PROF_AMAX, m->s_rs, ps->bytes);
      CUDA_CHECK(fsdpk::launch_amax(ps->tiles.d, ps->tiles.n, m->reg_acc, m->cfg, m->s_rs));
      pa.done();
    }
    if (comm_ready(m) && m->reg_size > 0) {
      // max of non-negative fp32 bit patterns == uint32 max (NaN patterns propagate)
      ProfScope pr(m, FSDP_PROF_ALL_REDUCE, m->s_rs, (int64_t)4 * m->reg_size);
      NCCL_CHECK(ncclAllReduce(m->reg_acc, m->reg_acc, (size_t)m->reg_size, ncclUint32, ncclMax, m->comm_rs, m->s_rs));
      pr.done();
    }
    {
      ProfScope pk(m, FSDP_PROF_SCALE, m->s_rs, (int64_t)ps->nidx * 12);
      if (history_len == 0) {
        CUDA_CHECK(fsdpk::launch_fp8_scale(ps->idx, ps->nidx, m->reg_acc, m->reg_amax, m->reg_scale, m->reg_elig,
                                           m->d_err, true, m->s_rs));
      } else {
        m->hist_len = history_len;
        CUDA_CHECK(fsdpk::launch_fp8_scale_delayed(ps->idx, ps->nidx, m->reg_acc, m->reg_amax, m->reg_scale,
                                                   m->reg_elig, m->reg_hist, m->reg_pos, m->reg_hinit, history_len,
                                                   kHistMax, m->d_err, m->s_rs));
      }
      pk.done();
    }
    CUDA_CHECK(cudaEventRecord(m->ev_pre_done, m->s_rs));
    CUDA_CHECK(cudaStreamWaitEvent(st, m->ev_pre_done, 0));
  });
}

fsdp_status_t fsdp_precompute_fp8_scales(fsdp_mesh_t* m, fsdp_layer_t* const* layers, int32_t n, void* stream) {
  return precompute_impl(m, layers, n, stream, 0);
}

fsdp_status_t fsdp_precompute_fp8_scales_delayed(fsdp_mesh_t* m, fsdp_layer_t* const* layers, int32_t n,
                                                 int32_t history_len, void* stream) {
  if (history_len < 1) {
    g_last_error = "history_len must be >= 1";
    return FSDP_ERR_INVALID_ARGUMENT;
  }
  return precompute_impl(m, layers, n, stream, history_len);
}

fsdp_status_t fsdp_fp8_scales(const fsdp_layer_t* l, const float** scales_dev, const float** amax_dev) {
  return guarded([&] {
    check_layer(l);
    if (scales_dev) *scales_dev = l->mesh->reg_scale + l->reg_base;
    if (amax_dev) *amax_dev = l->mesh->reg_amax + l->reg_base;
  });
}

// ------------------------------------------------------------------------- unshard
fsdp_status_t fsdp_unshard(fsdp_layer_t* l, fsdp_dtype_t dt, const float* scales, void* compute) {
  return guarded([&] {
    check_layer(l);
    fsdp_mesh* m = l->mesh;
    if (dt != FSDP_BFLOAT16 && dt != FSDP_FLOAT8_E4M3FN) fail(FSDP_ERR_DTYPE, "param_dtype must be BFLOAT16 or FLOAT8_E4M3FN");
    if (l->state != SHARDED) {
      // already unsharded (reshard_after_forward=False / the kept last block): a
      // no-op like FSDP2's unshard(), as long as the dtype matches
      if (dt != l->ushard_dtype) fail(FSDP_ERR_STATE, "layer is unsharded in another dtype (reshard it first)");
      return;
    }
    if (m->local && m->W > 1) fail(FSDP_ERR_UNAVAILABLE, "local mesh with world_size > 1 has no communicator");
    const bool fp8 = dt == FSDP_FLOAT8_E4M3FN;
    if (fp8 && !scales) scales = m->reg_scale + l->reg_base;
    DeviceGuard g(m->device);
    const int64_t sb = slot_bytes(l, fp8);
    const int64_t arena = fp8 ? l->L.arena_fp8 : l->L.arena_bf16;
    if (m->algo == FSDP_ALGO_P2P) {
      // fused path: ready handshake -> push (cast + store into every rank's arena) -> done
      SymSlot* ss = acquire_sym_slot(m, m->p2p_ag, (size_t)arena);
      const uint64_t epoch = ++ss->epoch;
      cudaStream_t cs = as_stream(compute);
      CUDA_CHECK(cudaEventRecord(l->ev_call, cs));
      CUDA_CHECK(cudaStreamWaitEvent(m->s_ag, l->ev_call, 0));
      if (ss->ever_used) CUDA_CHECK(cudaStreamWaitEvent(m->s_ag, ss->free_ev, 0));
      {
        ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_ag, 0);
        CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_AG_READY, ss->index), flag_local(m, FK_AG_READY, ss->index),
                                             m->W, m->rank, epoch, m->p2p_timeout_ns, m->d_err, m->s_ag));
        ph.done();
      }
      {
        const DevTiles& T = fp8 ? l->t_push_fp8 : l->t_push_bf16;
        ProfScope pp(m, FSDP_PROF_UNSHARD_PUSH, m->s_ag, fp8 ? l->push_bytes_fp8 : l->push_bytes_bf16);
        CUDA_CHECK(fsdpp::launch_unshard_push(T.d, T.n, l->shard, scales, peer_ptrs(m, ss->buf), m->W, m->rank,
                                              m->cfg, m->s_ag));
        pp.done();
      }
      {
        ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_ag, 0);
        CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_AG_DONE, ss->index), flag_local(m, FK_AG_DONE, ss->index),
                                             m->W, m->rank, epoch, m->p2p_timeout_ns, m->d_err, m->s_ag));
        ph.done();
      }
      CUDA_CHECK(cudaEventRecord(l->ev_done, m->s_ag));
      l->p2p_slot = ss;
      l->slot = nullptr;
      l->arena_base = ss->buf.local;
      l->ushard_dtype = dt;
      l->state = UNSHARDING;
      return;
    }
    if (m->W == 1) {
      // W = 1: the all-gather is the identity, so the unshard is ONE kernel that casts the
      // shard straight into the unsharded tensors (the push kernel with the local arena only)
      Slot* slot = acquire_slot(m, m->ag_slots, 0, (size_t)arena, 1);
      cudaStream_t cs = as_stream(compute);
      CUDA_CHECK(cudaEventRecord(l->ev_call, cs));
      CUDA_CHECK(cudaStreamWaitEvent(m->s_cin, l->ev_call, 0));
      if (slot->ever_used) CUDA_CHECK(cudaStreamWaitEvent(m->s_cin, slot->free_ev, 0));
      fsdpp::PeerPtrs pp{};
      pp.p[0] = (uint8_t*)slot->b.p;
      const DevTiles& T = fp8 ? l->t_push_fp8 : l->t_push_bf16;
      {
        ProfScope pc(m, FSDP_PROF_COPY_IN, m->s_cin, fp8 ? l->local_push_fp8 : l->local_push_bf16);
        fsdpk::LaunchCfg lcfg = m->cfg;   // W = 1: bulk stores too (0.915 vs 0.902 of HBM, r06)
        if (const char* e = std::getenv("FSDP_B200_W1_BULK")) if (std::atoi(e) == 0) lcfg.variant &= ~4;
        CUDA_CHECK(fsdpp::launch_unshard_push(T.d, T.n, l->shard, scales, pp, 1, 0, lcfg, m->s_cin));
        pc.done();
      }
      CUDA_CHECK(cudaEventRecord(l->ev_done, m->s_cin));
      l->slot = slot;
      l->p2p_slot = nullptr;
      l->arena_base = slot->b.p;
      l->ushard_dtype = dt;
      l->state = UNSHARDING;
      return;
    }
    Slot* slot = acquire_slot(m, m->ag_slots, (size_t)(m->W * sb), (size_t)arena, 1);
    cudaStream_t cs = as_stream(compute);
    // copy-in after the caller's prior work (optimizer step on the shard) and after the
    // previous user of this buffer released it
    CUDA_CHECK(cudaEventRecord(l->ev_call, cs));
    CUDA_CHECK(cudaStreamWaitEvent(m->s_cin, l->ev_call, 0));
    if (slot->ever_used) CUDA_CHECK(cudaStreamWaitEvent(m->s_cin, slot->free_ev, 0));
    uint8_t* ag = (uint8_t*)slot->a.p;
    do_copy_in(l, fp8, scales, ag + (size_t)m->rank * sb, m->s_cin);
    CUDA_CHECK(cudaEventRecord(l->ev_cin, m->s_cin));
    cudaEvent_t ready = l->ev_cin;
    if (comm_ready(m)) {
      CUDA_CHECK(cudaStreamWaitEvent(m->s_ag, l->ev_cin, 0));
      ProfScope pg(m, FSDP_PROF_ALL_GATHER, m->s_ag, (int64_t)(m->W - 1) * sb);
      NCCL_CHECK(ncclAllGather(ag + (size_t)m->rank * sb, ag, (size_t)sb, ncclUint8, m->comm_ag, m->s_ag));
      pg.done();
      CUDA_CHECK(cudaEventRecord(l->ev_ag, m->s_ag));
      ready = l->ev_ag;
    }
    CUDA_CHECK(cudaStreamWaitEvent(m->s_cout, ready, 0));
    std::vector<void*> outs(l->P);
    const auto& uoff = fp8 ? l->L.uoff_fp8 : l->L.uoff_bf16;
    for (int p = 0; p < l->P; ++p) outs[p] = (uint8_t*)slot->b.p + uoff[p];
    {
      ProfScope po(m, FSDP_PROF_COPY_OUT, m->s_cout, fp8 ? l->bytes_cout_fp8 : l->bytes_cout_bf16);
      launch_copy_out_all(l, fp8, ag, outs.data(), m->s_cout);
      po.done();
    }
    CUDA_CHECK(cudaEventRecord(l->ev_done, m->s_cout));
    l->slot = slot;
    l->p2p_slot = nullptr;
    l->arena_base = slot->b.p;
    l->ushard_dtype = dt;
    l->state = UNSHARDING;
  });
}

fsdp_status_t fsdp_wait_unshard(fsdp_layer_t* l, void* compute) {
  return guarded([&] {
    check_layer(l);
    if (l->state == UNSHARDED) return;
    if (l->state != UNSHARDING) fail(FSDP_ERR_STATE, "fsdp_wait_unshard without fsdp_unshard");
    DeviceGuard g(l->mesh->device);
    CUDA_CHECK(cudaStreamWaitEvent(as_stream(compute), l->ev_done, 0));
    l->state = UNSHARDED;
  });
}

fsdp_status_t fsdp_all_gather_params(fsdp_layer_t* l, fsdp_dtype_t dt, const float* scales, void* compute) {
  fsdp_status_t st = fsdp_unshard(l, dt, scales, compute);
  if (st != FSDP_OK) return st;
  return fsdp_wait_unshard(l, compute);
}

fsdp_status_t fsdp_unsharded_param(const fsdp_layer_t* l, int32_t p, void** dev, fsdp_dtype_t* dt) {
  return guarded([&] {
    check_layer(l);
    check_param(l, p);
    if (!dev) fail(FSDP_ERR_INVALID_ARGUMENT, "dev is NULL");
    if (l->state != UNSHARDED) fail(FSDP_ERR_STATE, "unsharded params are valid only between wait_unshard and reshard");
    const bool fp8 = l->ushard_dtype == FSDP_FLOAT8_E4M3FN;
    const auto& uoff = fp8 ? l->L.uoff_fp8 : l->L.uoff_bf16;
    *dev = (uint8_t*)l->arena_base + uoff[p];
    if (dt) *dt = (fp8 && l->L.fp8[p]) ? FSDP_FLOAT8_E4M3FN : FSDP_BFLOAT16;
  });
}

fsdp_status_t fsdp_reshard(fsdp_layer_t* l, void* compute) {
  return guarded([&] {
    check_layer(l);
    if (l->state == SHARDED) return;
    DeviceGuard g(l->mesh->device);
    cudaStream_t cs = as_stream(compute);
    if (l->state == UNSHARDING) CUDA_CHECK(cudaStreamWaitEvent(cs, l->ev_done, 0));
    // the buffer is free once everything enqueued on `compute` so far (the consumers of
    // the unsharded params) has run; the next user's copy-in waits on this event
    if (l->p2p_slot) {
      // peers write into this arena only after this rank's next ready handshake on it,
      // which the next unshard issues after waiting on free_ev
      CUDA_CHECK(cudaEventRecord(l->p2p_slot->free_ev, cs));
      l->p2p_slot->ever_used = true;
      l->p2p_slot->in_use = false;
      l->p2p_slot = nullptr;
    } else {
      release_slot(l->slot, cs);
    }
    l->slot = nullptr;
    l->arena_base = nullptr;
    l->state = SHARDED;
  });
}

// ------------------------------------------------------------------------- reduce-scatter
fsdp_status_t fsdp_reduce_scatter_grads(fsdp_layer_t* l, const void* const* grads, fsdp_dtype_t gd,
                                        fsdp_dtype_t rd, int32_t mean, int32_t accumulate, void* compute) {
  return guarded([&] {
    check_layer(l);
    fsdp_mesh* m = l->mesh;
    validate_grads(l, grads, gd, rd);
    if (l->rs_pending) fail(FSDP_ERR_STATE, "previous reduce_scatter_grads of this layer was not waited");
    if (m->local && m->W > 1) fail(FSDP_ERR_UNAVAILABLE, "local mesh with world_size > 1 has no communicator");
    DeviceGuard g(m->device);
    const bool obf = rd == FSDP_BFLOAT16;
    const int64_t osz = obf ? 2 : 4;
    const int64_t S = l->L.S;
    const bool hsdp = m->R > 1;            // + all-reduce across the replica group
    const int divisor = m->W * m->R;       // mean over every rank of the mesh
    // HSDP with accumulation: the shard-group result goes to a temp T, is all-reduced across
    // replicas, then added to the grad (the all-reduce must not see the old grad)
    const bool via_temp = hsdp && accumulate;
    cudaStream_t cs = as_stream(compute);
    auto replica_all_reduce = [&](float* buf) {
      ProfScope pa(m, FSDP_PROF_ALL_REDUCE, m->s_rs, (int64_t)2 * (m->R - 1) * S * 4 / m->R);
      NCCL_CHECK(ncclAllReduce(buf, buf, (size_t)S, ncclFloat32, ncclSum, m->comm_rep, m->s_rs));
      pa.done();
    };
    auto add_temp_into_grad = [&](const float* T) {
      ProfScope po(m, FSDP_PROF_RS_COPY_OUT, m->s_rs, S * 12);
      CUDA_CHECK(fsdpk::launch_rs_copy_out(T, false, l->grad, true, S, m->cfg, m->s_rs));
      po.done();
    };
    if (m->algo == FSDP_ALGO_P2P) {
      // fused path: stage the caller's grads into this rank's symmetric staging -> ready
      // handshake -> pull (every rank's rows of this rank, /divisor, ascending-rank fp32 sum,
      // written into the grad buffer) -> done handshake (staging reusable)
      const int64_t gsz = dtype_size(gd);
      // zero copy: the caller's grads already live in this layer's symmetric grad buffer
      bool zc = l->gbuf && l->gbuf_sym && gd == l->gbuf_dtype;
      for (int p = 0; zc && p < l->P; ++p)
        zc = l->L.numel[p] == 0 || grads[p] == (const void*)((uint8_t*)l->gbuf->buf.local + l->stg_off_el[p] * gsz);
      SymSlot* ss = nullptr;
      if (zc) {
        ss = l->gbuf;
      } else {
        const int prefer = (int)(m->rs_rr++ % 2);   // deterministic round robin: copy of i+1 overlaps pull of i
        ss = acquire_sym_slot(m, m->p2p_rs, (size_t)(l->stg_elems * gsz), prefer);
      }
      Slot* tmp = via_temp ? acquire_slot(m, m->rs_slots, 0, (size_t)(S * 4), 1) : nullptr;
      const uint64_t epoch = ++ss->epoch;
      CUDA_CHECK(cudaEventRecord(l->ev_rcall, cs));
      if (zc) {
        CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, l->ev_rcall, 0));
      } else {
        CUDA_CHECK(cudaStreamWaitEvent(m->s_rsc, l->ev_rcall, 0));
        if (ss->ever_used) CUDA_CHECK(cudaStreamWaitEvent(m->s_rsc, ss->free_ev, 0));
        {
          const DevTiles& T = gd == FSDP_BFLOAT16 ? l->t_stage_bf16 : l->t_stage_fp32;
          fsdpk::PtrArray pa{};
          for (int p = 0; p < l->P; ++p) pa.p[p] = grads[p];
          ProfScope pst(m, FSDP_PROF_STAGE_GRADS, m->s_rsc, 2 * l->grad_numel_total * gsz);
          CUDA_CHECK(fsdpp::launch_gather_copy(T.d, T.n, pa, ss->buf.local, m->cfg, m->s_rsc));
          pst.done();
        }
        CUDA_CHECK(cudaEventRecord(l->ev_k5, m->s_rsc));
        CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, l->ev_k5, 0));
      }
      float* target = l->grad;
      if (via_temp) {
        if (tmp->ever_used) CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, tmp->free_ev, 0));
        target = (float*)tmp->b.p;
        CUDA_CHECK(cudaMemsetAsync(target, 0, sizeof(float) * S, m->s_rs));   // padding stays 0
      }
      {
        ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_rs, 0);
        CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_READY, ss->index), flag_local(m, FK_RS_READY, ss->index),
                                             m->W, m->rank, epoch, m->p2p_timeout_ns, m->d_err, m->s_rs));
        ph.done();
      }
      {
        ProfScope pp(m, FSDP_PROF_RS_PULL, m->s_rs, (int64_t)(m->W - 1) * l->pull_elems * gsz);
        fsdpk::LaunchCfg pcfg = m->cfg;
        if (!zc) pcfg.variant &= ~2;   // bulk pull only without a concurrent staging copy (profiles/r06)
        CUDA_CHECK(fsdpp::launch_rs_pull(l->t_pull.d, l->t_pull.n, peer_ptrs(m, ss->buf), gd == FSDP_BFLOAT16, divisor,
                                         target, mean != 0, accumulate != 0 && !hsdp, obf, m->W, pcfg, m->s_rs));
        pp.done();
      }
      {
        ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_rs, 0);
        CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_DONE, ss->index), flag_local(m, FK_RS_DONE, ss->index),
                                             m->W, m->rank, epoch, m->p2p_timeout_ns, m->d_err, m->s_rs));
        ph.done();
      }
      CUDA_CHECK(cudaEventRecord(ss->free_ev, m->s_rs));
      ss->ever_used = true;
      ss->in_use = false;
      if (hsdp) {
        replica_all_reduce(target);
        if (via_temp) {
          add_temp_into_grad(target);
          release_slot(tmp, m->s_rs);
        }
      }
      CUDA_CHECK(cudaEventRecord(l->ev_rs_done, m->s_rs));
      l->rs_pending = true;
      return;
    }
    // NCCL path.  fp32 without accumulation: the reduce-scatter (or, at W=1, K5 itself)
    // writes straight into the layer's grad buffer — the zero-copy "view" copy-out
    const bool direct = !obf && !accumulate;
    const bool need_in = comm_ready(m) || !direct;
    const size_t stage_b = (comm_ready(m) && !direct) ? (size_t)(S * osz) : 0;
    Slot* slot = acquire_slot(m, m->rs_slots, need_in ? (size_t)(m->W * S * osz) : 0,
                              via_temp ? std::max(stage_b, (size_t)(S * 4)) : stage_b, 2);
    CUDA_CHECK(cudaEventRecord(l->ev_rcall, cs));
    CUDA_CHECK(cudaStreamWaitEvent(m->s_rsc, l->ev_rcall, 0));
    if (slot->ever_used) CUDA_CHECK(cudaStreamWaitEvent(m->s_rsc, slot->free_ev, 0));
    void* rs_in = need_in ? slot->a.p : (void*)l->grad;
    {
      ProfScope pk(m, FSDP_PROF_RS_COPY_IN, m->s_rsc,
                   l->grad_numel_total * dtype_size(gd) + (int64_t)m->W * S * osz);
      launch_rs_copy_in_all(l, grads, gd == FSDP_BFLOAT16, rs_in, obf, mean != 0, m->s_rsc);
      pk.done();
    }
    CUDA_CHECK(cudaEventRecord(l->ev_k5, m->s_rsc));
    CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, l->ev_k5, 0));
    const void* rs_out = rs_in;   // W == 1: the reduce-scatter is the identity
    if (comm_ready(m)) {
      void* out = direct ? (void*)l->grad : slot->b.p;
      ProfScope pr(m, FSDP_PROF_REDUCE_SCATTER, m->s_rs, (int64_t)(m->W - 1) * S * osz);
      NCCL_CHECK(ncclReduceScatter(rs_in, out, (size_t)S, obf ? ncclBfloat16 : ncclFloat32, ncclSum, m->comm_rs,
                                   m->s_rs));
      pr.done();
      rs_out = out;
    }
    if (via_temp) {
      // widen / copy the shard-group result into T (in place when it already is fp32 in
      // the staging buffer), all-reduce T across replicas, add T into the grad
      float* T = (float*)slot->b.p;
      if (rs_out != (const void*)T || obf) {
        ProfScope po(m, FSDP_PROF_RS_COPY_OUT, m->s_rs, S * (osz + 4));
        CUDA_CHECK(fsdpk::launch_rs_copy_out(rs_out, obf, T, false, S, m->cfg, m->s_rs));
        po.done();
      }
      replica_all_reduce(T);
      add_temp_into_grad(T);
    } else {
      if (!direct) {
        ProfScope po(m, FSDP_PROF_RS_COPY_OUT, m->s_rs, S * (osz + 4 + (accumulate ? 4 : 0)));
        CUDA_CHECK(fsdpk::launch_rs_copy_out(rs_out, obf, l->grad, accumulate != 0, S, m->cfg, m->s_rs));
        po.done();
      }
      if (hsdp) replica_all_reduce(l->grad);
    }
    CUDA_CHECK(cudaEventRecord(l->ev_rs_done, m->s_rs));
    release_slot(slot, m->s_rs);
    l->rs_pending = true;
  });
}

fsdp_status_t fsdp_wait_reduce_scatter(fsdp_layer_t* l, void* compute) {
  return guarded([&] {
    check_layer(l);
    if (!l->rs_pending) return;
    DeviceGuard g(l->mesh->device);
    CUDA_CHECK(cudaStreamWaitEvent(as_stream(compute), l->ev_rs_done, 0));
    l->rs_pending = false;
  });
}

fsdp_status_t fsdp_sharded_grad(const fsdp_layer_t* l, int32_t p, float** dev) {
  return guarded([&] {
    if (!l || !dev) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    check_param(l, p);
    *dev = l->grad + l->L.metas[p].elem_offset;
  });
}

fsdp_status_t fsdp_sharded_grad_flat(const fsdp_layer_t* l, float** dev) {
  return guarded([&] {
    if (!l || !dev) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    *dev = l->grad;
  });
}

fsdp_status_t fsdp_zero_grad(fsdp_layer_t* l, void* stream) {
  return guarded([&] {
    check_layer(l);
    DeviceGuard g(l->mesh->device);
    CUDA_CHECK(cudaMemsetAsync(l->grad, 0, sizeof(float) * (size_t)l->L.S, as_stream(stream)));
  });
}

// ------------------------------------------------------------------------- stage entry points
fsdp_status_t fsdp_stage_copy_in(const fsdp_layer_t* lc, fsdp_dtype_t dt, const float* scales, void* slot,
                                 void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    if (!slot) fail(FSDP_ERR_INVALID_ARGUMENT, "ag_slot is NULL");
    if (dt != FSDP_BFLOAT16 && dt != FSDP_FLOAT8_E4M3FN) fail(FSDP_ERR_DTYPE, "param_dtype must be BFLOAT16 or FLOAT8_E4M3FN");
    const bool fp8 = dt == FSDP_FLOAT8_E4M3FN;
    if (fp8 && !scales) scales = l->mesh->reg_scale + l->reg_base;
    DeviceGuard g(l->mesh->device);
    do_copy_in(l, fp8, scales, slot, as_stream(stream));
  });
}

fsdp_status_t fsdp_stage_copy_out(const fsdp_layer_t* lc, fsdp_dtype_t dt, const void* ag, void* const* outs,
                                  void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    if (!ag || !outs) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL buffer");
    for (int p = 0; p < l->P; ++p)
      if (!outs[p] && l->L.numel[p] > 0) fail(FSDP_ERR_INVALID_ARGUMENT, "full_out[p] is NULL");
    if (dt != FSDP_BFLOAT16 && dt != FSDP_FLOAT8_E4M3FN) fail(FSDP_ERR_DTYPE, "param_dtype must be BFLOAT16 or FLOAT8_E4M3FN");
    const bool fp8 = dt == FSDP_FLOAT8_E4M3FN;
    DeviceGuard g(l->mesh->device);
    ProfScope po(l->mesh, FSDP_PROF_COPY_OUT, as_stream(stream), fp8 ? l->bytes_cout_fp8 : l->bytes_cout_bf16);
    launch_copy_out_all(l, fp8, ag, outs, as_stream(stream));
    po.done();
  });
}

fsdp_status_t fsdp_stage_local_amax(const fsdp_layer_t* lc, float* amax_out, void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    if (!amax_out) fail(FSDP_ERR_INVALID_ARGUMENT, "amax_out is NULL");
    DeviceGuard g(l->mesh->device);
    cudaStream_t st = as_stream(stream);
    std::vector<Tile> tiles;
    fsdpl::append_tiles_amax(l->L, l->shard, 0, &tiles);
    DevTiles T;
    T.upload(tiles);   // synchronous upload (test entry point, not on the hot path)
    CUDA_CHECK(cudaMemsetAsync(amax_out, 0, sizeof(float) * l->P, st));
    cudaError_t e = fsdpk::launch_amax(T.d, T.n, reinterpret_cast<uint32_t*>(amax_out), l->mesh->cfg, st);
    CUDA_CHECK(cudaStreamSynchronize(st));
    T.release();
    CUDA_CHECK(e);
  });
}

fsdp_status_t fsdp_stage_fp8_scale(const fsdp_layer_t* lc, const float* amax, float* scale_out, void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    if (!amax || !scale_out) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL buffer");
    DeviceGuard g(l->mesh->device);
    // amax is read as non-negative fp32 bit patterns; amax_out == amax (rewritten as is)
    CUDA_CHECK(fsdpk::launch_fp8_scale(l->d_idx_local, l->P, (uint32_t*)const_cast<float*>(amax),
                                       const_cast<float*>(amax), scale_out, l->mesh->reg_elig + l->reg_base,
                                       l->mesh->d_err, false, as_stream(stream)));
  });
}

fsdp_status_t fsdp_stage_rs_copy_in(const fsdp_layer_t* lc, const void* const* grads, fsdp_dtype_t gd,
                                    fsdp_dtype_t rd, int32_t mean, void* rs_in, void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    validate_grads(l, grads, gd, rd);
    if (!rs_in) fail(FSDP_ERR_INVALID_ARGUMENT, "rs_in is NULL");
    DeviceGuard g(l->mesh->device);
    const int64_t osz = rd == FSDP_BFLOAT16 ? 2 : 4;
    ProfScope pk(l->mesh, FSDP_PROF_RS_COPY_IN, as_stream(stream),
                 l->grad_numel_total * dtype_size(gd) + (int64_t)l->mesh->W * l->L.S * osz);
    launch_rs_copy_in_all(l, grads, gd == FSDP_BFLOAT16, rs_in, rd == FSDP_BFLOAT16, mean != 0, as_stream(stream));
    pk.done();
  });
}

fsdp_status_t fsdp_stage_rs_copy_out(fsdp_layer_t* l, const void* rs_out, fsdp_dtype_t rd, int32_t accumulate,
                                     void* stream) {
  return guarded([&] {
    check_layer(l);
    if (!rs_out) fail(FSDP_ERR_INVALID_ARGUMENT, "rs_out is NULL");
    if (rd != FSDP_BFLOAT16 && rd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "reduce_dtype must be FLOAT32 or BFLOAT16");
    DeviceGuard g(l->mesh->device);
    const int64_t osz = rd == FSDP_BFLOAT16 ? 2 : 4;
    ProfScope po(l->mesh, FSDP_PROF_RS_COPY_OUT, as_stream(stream), l->L.S * (osz + 4 + (accumulate ? 4 : 0)));
    CUDA_CHECK(fsdpk::launch_rs_copy_out(rs_out, rd == FSDP_BFLOAT16, l->grad, accumulate != 0, l->L.S,
                                         l->mesh->cfg, as_stream(stream)));
    po.done();
  });
}

}  // extern "C"

// ------------------------------------------------------------------------- P2P stage entry points
extern "C" {

fsdp_status_t fsdp_unsharded_layout(const fsdp_layer_t* l, fsdp_dtype_t dt, int64_t* offsets, int64_t* total) {
  return guarded([&] {
    if (!l) fail(FSDP_ERR_INVALID_ARGUMENT, "layer is NULL");
    if (dt != FSDP_BFLOAT16 && dt != FSDP_FLOAT8_E4M3FN) fail(FSDP_ERR_DTYPE, "param_dtype must be BFLOAT16 or FLOAT8_E4M3FN");
    const bool fp8 = dt == FSDP_FLOAT8_E4M3FN;
    const auto& u = fp8 ? l->L.uoff_fp8 : l->L.uoff_bf16;
    if (offsets) std::copy(u.begin(), u.end(), offsets);
    if (total) *total = fp8 ? l->L.arena_fp8 : l->L.arena_bf16;
  });
}

fsdp_status_t fsdp_stage_unshard_push(const fsdp_layer_t* lc, fsdp_dtype_t dt, const float* scales,
                                      void* const* arenas, void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    fsdp_mesh* m = l->mesh;
    if (m->W > fsdpp::kMaxRanks) fail(FSDP_ERR_UNAVAILABLE, "world size above the P2P limit");
    if (!arenas) fail(FSDP_ERR_INVALID_ARGUMENT, "arenas is NULL");
    if (dt != FSDP_BFLOAT16 && dt != FSDP_FLOAT8_E4M3FN) fail(FSDP_ERR_DTYPE, "param_dtype must be BFLOAT16 or FLOAT8_E4M3FN");
    const bool fp8 = dt == FSDP_FLOAT8_E4M3FN;
    if (fp8 && !scales) scales = m->reg_scale + l->reg_base;
    fsdpp::PeerPtrs pp{};
    for (int r = 0; r < m->W; ++r) {
      if (!arenas[r]) fail(FSDP_ERR_INVALID_ARGUMENT, "arenas[r] is NULL");
      pp.p[r] = (uint8_t*)arenas[r];
    }
    DeviceGuard g(m->device);
    const DevTiles& T = fp8 ? l->t_push_fp8 : l->t_push_bf16;
    ProfScope ps(m, FSDP_PROF_UNSHARD_PUSH, as_stream(stream), fp8 ? l->push_bytes_fp8 : l->push_bytes_bf16);
    CUDA_CHECK(fsdpp::launch_unshard_push(T.d, T.n, l->shard, scales, pp, m->W, m->rank, m->cfg, as_stream(stream)));
    ps.done();
  });
}

fsdp_status_t fsdp_grad_staging_layout(const fsdp_layer_t* l, int64_t* offsets, int64_t* total) {
  return guarded([&] {
    if (!l) fail(FSDP_ERR_INVALID_ARGUMENT, "layer is NULL");
    if (offsets) std::copy(l->stg_off_el.begin(), l->stg_off_el.end(), offsets);
    if (total) *total = l->stg_elems;
  });
}

fsdp_status_t fsdp_stage_grads_to_staging(const fsdp_layer_t* lc, const void* const* grads, fsdp_dtype_t gd,
                                          void* staging, void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    validate_grads(l, grads, gd, FSDP_FLOAT32);
    if (!staging) fail(FSDP_ERR_INVALID_ARGUMENT, "staging is NULL");
    DeviceGuard g(l->mesh->device);
    const DevTiles& T = gd == FSDP_BFLOAT16 ? l->t_stage_bf16 : l->t_stage_fp32;
    fsdpk::PtrArray pa{};
    for (int p = 0; p < l->P; ++p) pa.p[p] = grads[p];
    ProfScope ps(l->mesh, FSDP_PROF_STAGE_GRADS, as_stream(stream), 2 * l->grad_numel_total * dtype_size(gd));
    CUDA_CHECK(fsdpp::launch_gather_copy(T.d, T.n, pa, staging, l->mesh->cfg, as_stream(stream)));
    ps.done();
  });
}

fsdp_status_t fsdp_stage_rs_pull(fsdp_layer_t* l, const void* const* stagings, fsdp_dtype_t gd, fsdp_dtype_t rd,
                                 int32_t mean, int32_t accumulate, void* stream) {
  return guarded([&] {
    check_layer(l);
    fsdp_mesh* m = l->mesh;
    if (m->W > 8) fail(FSDP_ERR_UNAVAILABLE, "the pull kernel supports W <= 8");
    if (!stagings) fail(FSDP_ERR_INVALID_ARGUMENT, "stagings is NULL");
    if (gd != FSDP_BFLOAT16 && gd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "grad_dtype must be BFLOAT16 or FLOAT32");
    if (rd != FSDP_BFLOAT16 && rd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "reduce_dtype must be FLOAT32 or BFLOAT16");
    fsdpp::PeerPtrs pp{};
    for (int r = 0; r < m->W; ++r) {
      if (!stagings[r]) fail(FSDP_ERR_INVALID_ARGUMENT, "stagings[r] is NULL");
      pp.p[r] = (uint8_t*)stagings[r];
    }
    DeviceGuard g(m->device);
    ProfScope ps(m, FSDP_PROF_RS_PULL, as_stream(stream), (int64_t)(m->W - 1) * l->pull_elems * dtype_size(gd));
    CUDA_CHECK(fsdpp::launch_rs_pull(l->t_pull.d, l->t_pull.n, pp, gd == FSDP_BFLOAT16, m->W * m->R, l->grad, mean != 0,
                                     accumulate != 0, rd == FSDP_BFLOAT16, m->W, m->cfg, as_stream(stream)));
    ps.done();
  });
}

fsdp_status_t fsdp_full_grad_buffer(fsdp_layer_t* l, fsdp_dtype_t gd, int32_t p, void** dev) {
  return guarded([&] {
    check_layer(l);
    check_param(l, p);
    if (!dev) fail(FSDP_ERR_INVALID_ARGUMENT, "dev is NULL");
    if (gd != FSDP_BFLOAT16 && gd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "grad_dtype must be BFLOAT16 or FLOAT32");
    fsdp_mesh* m = l->mesh;
    const int64_t gsz = dtype_size(gd);
    if (!l->gbuf) {
      DeviceGuard g(m->device);
      auto* s = new SymSlot();
      s->free_ev = new_event();
      const size_t bytes = (size_t)std::max<int64_t>(l->stg_elems, 128) * gsz;
      if (m->p2p_ok) {   // collective: every rank maps every peer's buffer
        if (kPoolSlots + m->gbuf_seq >= kFlagSlots) fail(FSDP_ERR_UNAVAILABLE, "too many layer grad buffers");
        s->index = kPoolSlots + m->gbuf_seq++;
        if (!sym_alloc(m, s->buf, bytes)) {
          cudaEventDestroy(s->free_ev);
          delete s;
          fail(FSDP_ERR_OUT_OF_MEMORY, "symmetric grad buffer allocation/mapping failed");
        }
        l->gbuf_sym = true;
      } else {
        CUDA_CHECK(cudaMalloc(&s->buf.local, bytes + 256));
        CUDA_CHECK(cudaMemset(s->buf.local, 0, bytes + 256));
        s->buf.bytes = bytes;
        l->gbuf_sym = false;
      }
      l->gbuf = s;
      l->gbuf_dtype = gd;
    } else if (gd != l->gbuf_dtype) {
      fail(FSDP_ERR_DTYPE, "the layer's grad buffer was created with another grad_dtype");
    }
    *dev = (uint8_t*)l->gbuf->buf.local + l->stg_off_el[p] * gsz;
  });
}

}  // extern "C"
