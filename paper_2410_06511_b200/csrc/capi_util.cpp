// Internal helpers of the C ABI: pools, registry, symmetric memory, launch wrappers.
#include "capi_internal.h"

namespace fsdpc {

thread_local std::string g_last_error;


cudaEvent_t new_event(bool timing) {
  cudaEvent_t e;
  CUDA_CHECK(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  return e;
}


// ---- profiling helpers

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
Slot* acquire_slot(fsdp_mesh* m, std::vector<Slot*>& pool, size_t a_bytes, size_t b_bytes, int min_slots,
                   const Capture& cap) {
  if (cap.on) {   // capturing: least recently used free slot that is big enough; no queries, no growth
    Slot* best = nullptr;
    for (Slot* s : pool)
      if (!s->in_use && s->a.cap >= a_bytes && s->b.cap >= b_bytes && (!best || s->last_use < best->last_use))
        best = s;
    if (!best)
      fail(FSDP_ERR_STATE, "no warm buffer for this call inside a CUDA graph capture: run the same step once "
                           "eagerly before capturing it");
    best->in_use = true;
    best->last_use = ++m->use_seq;
    return best;
  }
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
    best->a.ensure(a_bytes, m->allocator);
    best->b.ensure(b_bytes, m->allocator);
  }
  best->in_use = true;
  best->last_use = ++m->use_seq;
  return best;
}

template <class SlotT>
static void release_any(SlotT* s, cudaStream_t last_user, const Capture& cap) {
  if (cap.on) {
    if (!s->cap_ev) s->cap_ev = new_event();
    CUDA_CHECK(cudaEventRecord(s->cap_ev, last_user));
    s->ev_capture = cap.id;
  } else {
    CUDA_CHECK(cudaEventRecord(s->free_ev, last_user));
    s->ev_capture = 0;
  }
  s->ever_used = true;
  s->in_use = false;
}

void release_slot(Slot* s, cudaStream_t last_user, const Capture& cap) { release_any(s, last_user, cap); }
void release_sym_slot(SymSlot* s, cudaStream_t last_user, const Capture& cap) { release_any(s, last_user, cap); }

void check_mesh(const fsdp_mesh* m) {
  if (!m) fail(FSDP_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (m->aborted) fail(m->abort_status, "mesh aborted earlier: " + m->abort_msg);
}

void abort_mesh(fsdp_mesh* m, fsdp_status_t st, const std::string& msg) {
  if (!m->aborted) {   // the first reason sticks
    m->aborted = true;
    m->abort_status = st;
    m->abort_msg = msg;
  }
  fail(st, msg);
}
void check_layer(const fsdp_layer* l) {
  if (!l) fail(FSDP_ERR_INVALID_ARGUMENT, "layer is NULL");
  check_mesh(l->mesh);
}
void check_param(const fsdp_layer* l, int p) {
  if (p < 0 || p >= l->P) fail(FSDP_ERR_INVALID_ARGUMENT, "param index out of range");
}

bool comm_ready(const fsdp_mesh* m) { return !m->local && m->W > 1; }
bool nccl_ok(const fsdp_mesh* m) { return !m->local && !m->hc_fn && (m->W > 1 || m->R > 1); }

// fp8 registry: fixed capacity, allocated once per mesh, so the device pointers handed out by
// fsdp_fp8_scales (and baked into captured CUDA graphs) stay valid for the mesh's lifetime.
// Entries are assigned in fsdp_shard order (a collective call, so every rank assigns alike)
// and are recycled only once every layer of the mesh has been destroyed.
void registry_init(fsdp_mesh* m) {
  int cap = kRegCapDefault;
  if (const char* e = std::getenv("FSDP_B200_REGISTRY_CAP")) cap = std::max(64, std::min(1 << 22, std::atoi(e)));
  CUDA_CHECK(cudaMalloc(&m->reg_acc, sizeof(uint32_t) * cap));
  CUDA_CHECK(cudaMalloc(&m->reg_amax, sizeof(float) * cap));
  CUDA_CHECK(cudaMalloc(&m->reg_scale, sizeof(float) * cap));
  CUDA_CHECK(cudaMalloc(&m->reg_elig, cap));
  CUDA_CHECK(cudaMalloc(&m->reg_pos, sizeof(int32_t) * cap));
  CUDA_CHECK(cudaMalloc(&m->reg_hinit, cap));
  CUDA_CHECK(cudaMemset(m->reg_acc, 0, sizeof(uint32_t) * cap));
  CUDA_CHECK(cudaMemset(m->reg_amax, 0, sizeof(float) * cap));
  CUDA_CHECK(cudaMemset(m->reg_scale, 0, sizeof(float) * cap));
  CUDA_CHECK(cudaMemset(m->reg_elig, 0, cap));
  CUDA_CHECK(cudaMemset(m->reg_pos, 0, sizeof(int32_t) * cap));
  CUDA_CHECK(cudaMemset(m->reg_hinit, 0, cap));
  m->reg_cap = cap;
}

int registry_reserve(fsdp_mesh* m, int n) {
  if (m->layers.empty() && m->reg_size > 0) {   // every layer destroyed: start over
    CUDA_CHECK(cudaDeviceSynchronize());
    CUDA_CHECK(cudaMemset(m->reg_acc, 0, sizeof(uint32_t) * m->reg_size));
    CUDA_CHECK(cudaMemset(m->reg_amax, 0, sizeof(float) * m->reg_size));
    CUDA_CHECK(cudaMemset(m->reg_scale, 0, sizeof(float) * m->reg_size));
    CUDA_CHECK(cudaMemset(m->reg_elig, 0, m->reg_size));
    CUDA_CHECK(cudaMemset(m->reg_pos, 0, sizeof(int32_t) * m->reg_size));
    CUDA_CHECK(cudaMemset(m->reg_hinit, 0, m->reg_size));
    m->reg_size = 0;
  }
  if (m->reg_size + n > m->reg_cap)
    fail(FSDP_ERR_UNAVAILABLE, "fp8 registry full (" + std::to_string(m->reg_cap) +
                                   " params per mesh; raise FSDP_B200_REGISTRY_CAP)");
  const int base = m->reg_size;
  m->reg_size += n;
  return base;
}

// the delayed-scaling amax history [reg_cap][kHistMax], allocated at the first delayed
// precompute (16 MB at the default capacity) and never moved afterwards
void registry_ensure_hist(fsdp_mesh* m) {
  if (m->reg_hist) return;
  const size_t bytes = sizeof(float) * (size_t)m->reg_cap * kHistMax;
  CUDA_CHECK(cudaMalloc(&m->reg_hist, bytes));
  CUDA_CHECK(cudaMemset(m->reg_hist, 0, bytes));
}

void clear_presets(fsdp_mesh* m) {
  for (auto* ps : m->presets) { ps->tiles.release(); cudaFree(ps->idx); delete ps; }
  m->presets.clear();
}

int64_t dtype_size(fsdp_dtype_t d) { return d == FSDP_FLOAT32 ? 4 : (d == FSDP_BFLOAT16 ? 2 : 1); }

// ---- symmetric memory over CUDA IPC (collective helpers; every rank calls them in the
// same order, which the deterministic FSDP call sequence guarantees)
Group group_of(const fsdp_mesh* m, int grp) {
  if (grp == GRP_WORLD) return Group{m->comm_world, m->W * m->R, m->rep * m->W + m->rank};
  return Group{m->comm_ag, m->W, m->rank};
}

void group_allgather_host(fsdp_mesh* m, int grp, const void* send, void* recv, size_t bytes) {
  const Group G = group_of(m, grp);
  if (m->hc_fn) {   // the caller's host all-gather runs over the whole world: keep the group's part
    const int Wt = m->W * m->R;
    std::vector<uint8_t> all((size_t)Wt * bytes);
    if (m->hc_fn(send, all.data(), (int64_t)bytes, m->hc_ctx) != 0)
      fail(FSDP_ERR_UNAVAILABLE, "host all-gather callback failed");
    for (int q = 0; q < G.W; ++q) {
      const int g = grp == GRP_WORLD ? q : m->rep * m->W + q;
      std::memcpy((uint8_t*)recv + (size_t)q * bytes, all.data() + (size_t)g * bytes, bytes);
    }
    return;
  }
  uint8_t* d = nullptr;
  CUDA_CHECK(cudaMalloc(&d, bytes * G.W));
  CUDA_CHECK(cudaMemcpy(d + bytes * G.rank, send, bytes, cudaMemcpyHostToDevice));
  NCCL_CHECK(ncclAllGather(d + bytes * G.rank, d, bytes, ncclUint8, G.comm, m->s_ag));
  CUDA_CHECK(cudaStreamSynchronize(m->s_ag));
  CUDA_CHECK(cudaMemcpy(recv, d, bytes * G.W, cudaMemcpyDeviceToHost));
  cudaFree(d);
}

void mesh_barrier(fsdp_mesh* m, int grp) {
  if (m->hc_fn) {
    const uint8_t one = 1;
    std::vector<uint8_t> all(group_of(m, grp).W);
    group_allgather_host(m, grp, &one, all.data(), 1);
    return;
  }
  const Group g = group_of(m, grp);
  NCCL_CHECK(ncclAllReduce(m->d_barrier, m->d_barrier, 1, ncclInt32, ncclSum, g.comm, m->s_ag));
  CUDA_CHECK(cudaStreamSynchronize(m->s_ag));
}

// all ranks of the group agree that `ok` holds everywhere
bool mesh_all_ok(fsdp_mesh* m, bool ok, int grp) {
  if (m->hc_fn) {
    const uint8_t v = ok ? 1 : 0;
    std::vector<uint8_t> all(group_of(m, grp).W);
    group_allgather_host(m, grp, &v, all.data(), 1);
    for (uint8_t x : all)
      if (!x) return false;
    return true;
  }
  const Group g = group_of(m, grp);
  int v = ok ? 1 : 0;
  CUDA_CHECK(cudaMemcpy(m->d_barrier, &v, sizeof(int), cudaMemcpyHostToDevice));
  NCCL_CHECK(ncclAllReduce(m->d_barrier, m->d_barrier, 1, ncclInt32, ncclMin, g.comm, m->s_ag));
  CUDA_CHECK(cudaStreamSynchronize(m->s_ag));
  CUDA_CHECK(cudaMemcpy(&v, m->d_barrier, sizeof(int), cudaMemcpyDeviceToHost));
  return v == 1;
}

// Rank-local (aborted mesh): unmap the peers' copies and free the local one, no barrier.
void sym_free_local(fsdp_mesh* m, SymBuf& b) {
  const Group g = group_of(m, b.grp);
  for (int r = 0; r < g.W; ++r)
    if (r != g.rank && r < (int)b.peers.size() && b.peers[r]) cudaIpcCloseMemHandle(b.peers[r]);
  if (b.local) cudaFree(b.local);
  cudaGetLastError();
  b = SymBuf();
}

// Collective over b's group: unmap the peers' copies, wait until every rank did, then free
// the local one.
void sym_free(fsdp_mesh* m, SymBuf& b) {
  const Group g = group_of(m, b.grp);
  for (int r = 0; r < g.W; ++r)
    if (r != g.rank && r < (int)b.peers.size() && b.peers[r]) cudaIpcCloseMemHandle(b.peers[r]);
  cudaGetLastError();
  mesh_barrier(m, b.grp);
  if (b.local) cudaFree(b.local);
  b = SymBuf();
}

// Returns false (on every rank of the group) if any rank failed to allocate or map.
bool sym_alloc(fsdp_mesh* m, SymBuf& b, size_t bytes, int grp) {
  const Group G = group_of(m, grp);
  b.grp = grp;
  bool ok = cudaMalloc(&b.local, bytes + 256) == cudaSuccess;
  cudaIpcMemHandle_t h{};
  if (ok) ok = cudaMemset(b.local, 0, bytes + 256) == cudaSuccess;
  if (ok) ok = cudaIpcGetMemHandle(&h, b.local) == cudaSuccess;
  cudaGetLastError();
  std::vector<cudaIpcMemHandle_t> hs(G.W);
  group_allgather_host(m, grp, &h, hs.data(), sizeof(h));
  b.peers.assign(G.W, nullptr);
  b.bytes = bytes;
  if (ok) {
    b.peers[G.rank] = b.local;
    for (int r = 0; r < G.W && ok; ++r) {
      if (r == G.rank) continue;
      void* p = nullptr;
      ok = cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      cudaGetLastError();
      b.peers[r] = ok ? p : nullptr;
    }
  }
  if (!mesh_all_ok(m, ok, grp)) {
    sym_free(m, b);
    return false;
  }
  return true;
}

fsdpp::FlagPtrs flag_remote(fsdp_mesh* m, int kind, int slot, int grp) {
  fsdpp::FlagPtrs f{};
  const SymBuf& fl = grp == GRP_WORLD ? m->wflags : m->flags;
  const size_t off = ((size_t)kind * kFlagSlots + slot) * fsdpp::kMaxRanks;
  for (int r = 0; r < (int)fl.peers.size(); ++r) f.p[r] = (unsigned long long*)fl.peers[r] + off;
  return f;
}
unsigned long long* flag_local(fsdp_mesh* m, int kind, int slot, int grp) {
  const SymBuf& fl = grp == GRP_WORLD ? m->wflags : m->flags;
  return (unsigned long long*)fl.local + ((size_t)kind * kFlagSlots + slot) * fsdpp::kMaxRanks;
}
unsigned long long* epoch_ctr(fsdp_mesh* m, int kind, int slot, int grp) {
  return (grp == GRP_WORLD ? m->d_wepochs : m->d_epochs) + (size_t)kind * kFlagSlots + slot;
}

// Deterministic choice: the lowest-index free slot (same on every rank, since in_use
// depends only on the call sequence); grows / creates slots collectively — except while
// capturing a CUDA graph, where the pool must already be warm.
SymSlot* acquire_sym_slot(fsdp_mesh* m, std::vector<SymSlot*>& pool, size_t bytes, int prefer, const Capture& cap,
                          int grp) {
  if (cap.on) {
    SymSlot* s = nullptr;
    if (prefer >= 0 && prefer < (int)pool.size() && !pool[prefer]->in_use && pool[prefer]->buf.bytes >= bytes)
      s = pool[prefer];
    for (size_t i = 0; !s && i < pool.size(); ++i)
      if (!pool[i]->in_use && pool[i]->buf.bytes >= bytes) s = pool[i];
    if (!s)
      fail(FSDP_ERR_STATE, "no warm symmetric buffer for this call inside a CUDA graph capture: run the same "
                           "step once eagerly before capturing it");
    s->in_use = true;
    return s;
  }
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
    mesh_barrier(m, grp);
    if (s->buf.local || !s->buf.peers.empty()) sym_free(m, s->buf);
    if (!sym_alloc(m, s->buf, bytes, grp)) fail(FSDP_ERR_OUT_OF_MEMORY, "symmetric buffer allocation/mapping failed");
  }
  s->in_use = true;
  return s;
}

fsdpp::PeerPtrs peer_ptrs(const fsdp_mesh*, const SymBuf& b) {   // indexed by rank in b's group
  fsdpp::PeerPtrs p{};
  for (int r = 0; r < (int)b.peers.size(); ++r) p.p[r] = (uint8_t*)b.peers[r];
  return p;
}

void p2p_teardown(fsdp_mesh* m) {
  if (m->hsdp_p2p) {   // world group first (its barrier covers every rank)
    CUDA_CHECK(cudaDeviceSynchronize());
    mesh_barrier(m, GRP_WORLD);
    for (SymSlot* s : m->p2p_wrs) {
      if (s->buf.local || !s->buf.peers.empty()) sym_free(m, s->buf);
      if (s->free_ev) cudaEventDestroy(s->free_ev);
      if (s->cap_ev) cudaEventDestroy(s->cap_ev);
      delete s;
    }
    m->p2p_wrs.clear();
    sym_free(m, m->wflags);
    m->hsdp_p2p = m->hsdp_rs_p2p = false;
  }
  if (!m->p2p_ok) return;
  CUDA_CHECK(cudaDeviceSynchronize());
  mesh_barrier(m);   // every rank's kernels are done with every peer buffer
  for (auto* pool : {&m->p2p_ag, &m->p2p_rs}) {
    for (SymSlot* s : *pool) {
      if (s->buf.local || !s->buf.peers.empty()) sym_free(m, s->buf);
      if (s->free_ev) cudaEventDestroy(s->free_ev);
      if (s->cap_ev) cudaEventDestroy(s->cap_ev);
      delete s;
    }
    pool->clear();
  }
  if (m->amax_sym.local) sym_free(m, m->amax_sym);
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

void do_copy_in(fsdp_layer* l, bool fp8, const float* scales, void* dst, cudaStream_t st, uint32_t* amax_acc) {
  fsdp_mesh* m = l->mesh;
  ProfScope ps(m, FSDP_PROF_COPY_IN, st, cin_bytes(l, fp8));
  if (fp8) CUDA_CHECK(fsdpk::launch_copy_in_fp8(l->t_cin_fp8.d, l->t_cin_fp8.n, l->shard, dst, scales, m->cfg, st,
                                                amax_acc));
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

// SURVEY §8(b) "NCCL async errors and timeouts are reported by wait_*": what has already
// happened on the device (a P2P handshake that gave up) or in NCCL is reported by the next
// wait_* call, without a sync; fsdp_mesh_synchronize drains and reports everything.
void poll_async_errors(fsdp_mesh* m) {
  const int err = *m->h_err;
  if ((err & 0xFF) == 2)
    abort_mesh(m, FSDP_ERR_TIMEOUT, "P2P handshake timed out waiting for shard rank " + std::to_string(err >> 8) +
                                        " (a rank skipped or diverged from the collective call sequence); mesh aborted");
  if (nccl_ok(m)) {
    for (ncclComm_t c : {m->comm_ag, m->comm_rs}) {
      ncclResult_t ar = ncclSuccess;
      if (c && ncclCommGetAsyncError(c, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
        abort_mesh(m, FSDP_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(ar));
    }
  }
}

void p2p_amax_allreduce(fsdp_mesh* m, int n, cudaStream_t st) {
  if (n <= 0) return;
  CUDA_CHECK(cudaMemcpyAsync(m->amax_sym.local, m->reg_acc, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToDevice, st));
  CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_READY, kAmaxSlot), flag_local(m, FK_RS_READY, kAmaxSlot),
                                       m->W, m->rank, epoch_ctr(m, FK_RS_READY, kAmaxSlot), m->p2p_timeout_ns,
                                       m->d_err, st, false, /*fence: the amax copy*/ true));
  CUDA_CHECK(fsdpp::launch_amax_max(peer_ptrs(m, m->amax_sym), m->W, m->reg_acc, n, st));
  // every rank has read every copy before any rank overwrites its own at the next call
  CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_DONE, kAmaxSlot), flag_local(m, FK_RS_DONE, kAmaxSlot),
                                       m->W, m->rank, epoch_ctr(m, FK_RS_DONE, kAmaxSlot), m->p2p_timeout_ns,
                                       m->d_err, st, m->cfg.pdl));
}

void ensure_pieces(fsdp_layer* l, int R) {
  if (l->piece_R == R) return;
  const std::vector<Tile> pull = fsdpl::tiles_pull(l->L, l->stg_off_el);
  int64_t P = 0;
  const std::vector<Tile> all = fsdpl::split_pieces(pull, l->L.S, R, &P);
  for (auto& t : l->t_piece) t.release();
  l->t_piece.assign(R, DevTiles());
  std::vector<std::vector<Tile>> per(R);
  for (const Tile& t : all) per[t.pad].push_back(t);
  for (int q = 0; q < R; ++q) l->t_piece[q].upload(per[q]);
  // gather tiles: src = dst (the piece sits at the grad's offsets in every result buffer),
  // merged round robin over the pieces starting after this replica's own, so the persistent
  // grid reads from every replica at once and the replicas start on different sources (a
  // piece-major order had every rank reading the same replica first: 530 GB/s, skewed ranks)
  std::vector<Tile> g;
  g.reserve(all.size());
  std::vector<size_t> pos(R, 0);
  const int rep = l->mesh->R == R ? l->mesh->rep : 0;
  for (bool more = true; more;) {
    more = false;
    for (int i = 1; i <= R; ++i) {
      const int q = (rep + i) % R;
      if (pos[q] < per[q].size()) {
        Tile t = per[q][pos[q]++];
        t.src = t.dst;
        g.push_back(t);
        more = true;
      }
    }
  }
  l->t_gather.upload(g);
  l->piece_R = R;
}

void ce_unshard(fsdp_layer* l, bool fp8, const float* scales, const fsdpp::PeerPtrs& arenas, cudaStream_t st,
                uint32_t* amax_acc) {
  fsdp_mesh* m = l->mesh;
  const fsdpl::Layout& L = l->L;
  const DevTiles& T = fp8 ? l->t_push_fp8 : l->t_push_bf16;
  const std::vector<int>& toff = fp8 ? l->push_tile_off_fp8 : l->push_tile_off_bf16;
  const std::vector<int64_t>& uoff = fp8 ? L.uoff_fp8 : L.uoff_bf16;
  fsdpp::PeerPtrs loc{};
  loc.p[0] = arenas.p[L.rank];
  fsdpk::LaunchCfg cfg = m->cfg;
  cfg.pdl = false;
  for (int p = 0; p < l->P; ++p) {
    const int nt = toff[p + 1] - toff[p];
    if (nt == 0) continue;
    CUDA_CHECK(fsdpp::launch_unshard_push(T.d + toff[p], nt, l->shard, scales, loc, 1, 0, cfg, st, amax_acc));
    CUDA_CHECK(cudaEventRecord(m->ev_ce, st));
    CUDA_CHECK(cudaStreamWaitEvent(m->s_ce, m->ev_ce, 0));
    const auto& mt = L.metas[p];
    const int64_t es = (fp8 && L.fp8[p]) ? 1 : 2;
    const int64_t off = uoff[p] + mt.row_begin * mt.rest * es;
    const size_t bytes = (size_t)(mt.row_count * mt.rest * es);
    for (int k = 1; k < L.W; ++k) {
      const int q = (L.rank + k) % L.W;
      CUDA_CHECK(cudaMemcpyAsync(arenas.p[q] + off, arenas.p[L.rank] + off, bytes, cudaMemcpyDeviceToDevice, m->s_ce));
    }
  }
  CUDA_CHECK(cudaEventRecord(m->ev_ce, m->s_ce));
  CUDA_CHECK(cudaStreamWaitEvent(st, m->ev_ce, 0));
}

void ce_scatter(fsdp_layer* l, const void* const* grads, int64_t gsz, const fsdpp::PeerPtrs& recvs, cudaStream_t st,
                bool include_self) {
  const fsdpl::Layout& L = l->L;
  for (int k = include_self ? 0 : 1; k < L.W; ++k) {
    const int r = (L.rank + k) % L.W;
    for (int p = 0; p < l->P; ++p) {
      const auto& mt = L.metas[p];
      const int64_t b = std::min<int64_t>((int64_t)r * mt.chunk_rows, mt.dim0);
      const int64_t e = std::min<int64_t>((int64_t)(r + 1) * mt.chunk_rows, mt.dim0);
      if (e <= b || mt.rest == 0) continue;
      const uint8_t* src = static_cast<const uint8_t*>(grads[p]) + (size_t)(b * mt.rest * gsz);
      uint8_t* dst = recvs.p[r] + (size_t)(((int64_t)L.rank * L.S + mt.elem_offset) * gsz);
      CUDA_CHECK(cudaMemcpyAsync(dst, src, (size_t)((e - b) * mt.rest * gsz), cudaMemcpyDeviceToDevice, st));
    }
  }
}

}  // namespace fsdpc
