// C ABI, part 1: errors, host layout, NCCL unique id, mesh lifecycle (init / HSDP / abort /
// destroy), algo selection, synchronize, profiling.  (Part 2: capi_layer.cpp, part 3:
// capi_stage.cpp, shared internals: capi_internal.h / capi_util.cpp.)
//
// Stream topology per mesh (all high priority, non-blocking):
//   NCCL mode                                    P2P mode (fused kernels)
//   s_cin  : K2/K3 copy-in; W=1 push             s_ag  : ready handshake -> push -> done
//   s_ag   : NCCL all-gather on comm_ag          s_rsc : grad staging copy (non zero-copy)
//   s_cout : K4 copy-out                         s_rs  : ready -> pull -> done handshakes,
//   s_rsc  : K5 RS copy-in                               replica all-reduce (HSDP)
//   s_rs   : NCCL reduce-scatter / all-reduce(max), K6, K1, K1b
// The unshard of unit i+1 runs while unit i's reduce-scatter is in flight (two comms in
// NCCL mode; separate streams and flag arrays in P2P mode).  Buffer reuse is guarded by
// CUDA events recorded on the consuming stream and, across GPUs, by epoch flags — never
// record_stream — so memory is released deterministically.
#include "capi_internal.h"

using namespace fsdpc;

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
  for (cudaStream_t* s : {&m->s_cin, &m->s_ag, &m->s_cout, &m->s_rsc, &m->s_rs, &m->s_ce})
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
  m->cfg.variant = 78;   // + 64: the W=1 bf16 unshard as the TMA-in/TMA-out cast (profiles/round2/r2cast)
  if (const char* e = std::getenv("FSDP_B200_VARIANT")) m->cfg.variant = std::atoi(e);
  if (const char* e = std::getenv("FSDP_B200_PULL_CHUNK")) {
    const int c = std::atoi(e);
    if (c >= 1024 && c <= 16384 && (c & (c - 1)) == 0) m->cfg.pull_chunk = c;
  }
  if (const char* e = std::getenv("FSDP_B200_PULL_STAGES")) m->cfg.pull_stages = std::max(2, std::min(4, std::atoi(e)));
  if (const char* e = std::getenv("FSDP_B200_PDL")) m->cfg.pdl = std::atoi(e) != 0;
  if (const char* e = std::getenv("FSDP_B200_K5_STAGES")) m->cfg.k5_stages = std::max(2, std::min(4, std::atoi(e)));
  m->cfg.grid_cap = sms * (per_sm > 0 ? per_sm : 4);
  // device error flag in mapped pinned host memory: kernels store a code (plain stores, no
  // atomics over PCIe), the host reads it without a copy or sync (wait_* poll it)
  void* herr = nullptr;
  CUDA_CHECK(cudaHostAlloc(&herr, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
  m->h_err = static_cast<volatile int*>(herr);
  *m->h_err = 0;
  void* derr = nullptr;
  CUDA_CHECK(cudaHostGetDevicePointer(&derr, herr, 0));
  m->d_err = static_cast<int*>(derr);
  m->ev_ce = new_event();
  m->ev_pre_call = new_event();
  m->ev_pre_done = new_event();
  CUDA_CHECK(cudaMalloc(&m->d_barrier, sizeof(int)));
  CUDA_CHECK(cudaMemset(m->d_barrier, 0, sizeof(int)));
  registry_init(m);
}

// P2P capability: W in [2, 8] and every rank can map every peer's buffer (collective).
static void p2p_init(fsdp_mesh* m) {
  if (const char* e = std::getenv("FSDP_B200_STORE_OWN")) m->store_own_direct = std::atoi(e) != 0;
  if (const char* e = std::getenv("FSDP_B200_AMAX_FUSE")) m->amax_fuse = std::atoi(e) != 0;
  if (const char* e = std::getenv("FSDP_B200_CE")) m->ce = std::atoi(e) != 0;
  if (m->local) return;
  const size_t fbytes = sizeof(unsigned long long) * FK_NUM * kFlagSlots * fsdpp::kMaxRanks;
  const size_t ebytes = sizeof(unsigned long long) * FK_NUM * kFlagSlots;
  const char* env = std::getenv("FSDP_B200_ALGO");
  const bool want_nccl = env && std::string(env) == "nccl";
  // HSDP on one NVSwitch domain: world-group symmetric memory for the reduce-scatter pull
  // (collective over the world; the same decision on every rank: R, W and the environment)
  if (m->R > 1 && m->W * m->R <= 8 && (m->comm_world || m->hc_fn)) {
    // two-phase moves fewer bytes iff (RW-1) 2/R + (R-1) 4/R < (RW-1) 2, i.e. R W > 3
    m->hsdp_two_phase = m->W * m->R > 3;
    if (const char* e = std::getenv("FSDP_B200_HSDP_RS")) m->hsdp_two_phase = m->hsdp_two_phase && std::atoi(e) != 1;
    const char* h = std::getenv("FSDP_B200_HSDP_P2P");
    if (!(h && std::atoi(h) == 0)) {
      m->hsdp_p2p = sym_alloc(m, m->wflags, fbytes, GRP_WORLD);
      if (m->hsdp_p2p) {
        CUDA_CHECK(cudaMalloc(&m->d_wepochs, ebytes));
        CUDA_CHECK(cudaMemset(m->d_wepochs, 0, ebytes));
      }
      m->hsdp_rs_p2p = m->hsdp_p2p && !want_nccl;
    }
  }
  if (m->W < 2 || m->W > 8) return;
  m->p2p_ok = sym_alloc(m, m->flags, fbytes);
  if (m->p2p_ok && !sym_alloc(m, m->amax_sym, sizeof(uint32_t) * (size_t)std::max(m->reg_cap, 1))) {
    sym_free(m, m->flags);
    m->p2p_ok = false;
  }
  CUDA_CHECK(cudaMalloc(&m->d_epochs, ebytes));
  CUDA_CHECK(cudaMemset(m->d_epochs, 0, ebytes));
  m->algo = (m->p2p_ok && !want_nccl) ? FSDP_ALGO_P2P : FSDP_ALGO_NCCL;
  if (const char* t = std::getenv("FSDP_B200_P2P_TIMEOUT_MS"))
    m->p2p_timeout_ns = (unsigned long long)std::max(1L, std::atol(t)) * 1000000ull;
  if (const char* e = std::getenv("FSDP_B200_REDUCE_CTAS_PER_SM")) m->reduce_per_sm = std::max(0, std::min(16, std::atoi(e)));
  if (const char* e = std::getenv("FSDP_B200_GATHER_CTAS_PER_SM")) m->gather_per_sm = std::max(0, std::min(16, std::atoi(e)));
  if (const char* r = std::getenv("FSDP_B200_P2P_RS"))
    m->p2p_rs_mode = std::string(r) == "pull" ? FSDP_P2P_RS_PULL
                     : std::string(r) == "store" ? FSDP_P2P_RS_STORE : FSDP_P2P_RS_AUTO;
}

static fsdp_status_t mesh_init_impl(const uint8_t* id, int32_t W, int32_t rank, int32_t dev, bool local,
                                    fsdp_mesh_t** out, int32_t shard_size = 0,
                                    fsdp_host_allgather_fn hc_fn = nullptr, void* hc_ctx = nullptr) {
  return guarded([&] {
    if (!out) fail(FSDP_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (W < 1 || rank < 0 || rank >= W) fail(FSDP_ERR_INVALID_ARGUMENT, "invalid world_size/rank");
    if (!local && !id && !hc_fn) fail(FSDP_ERR_INVALID_ARGUMENT, "unique id is NULL");
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
    m->hc_fn = hc_fn;
    m->hc_ctx = hc_ctx;
    try {
      mesh_common_init(m);
      if (hc_fn) {   // host-collective P2P mesh: no NCCL (header: fsdp_mesh_init_hostcoll)
        p2p_init(m);
        if (m->W > 1 && !m->p2p_ok) fail(FSDP_ERR_UNAVAILABLE, "host-collective mesh: a rank cannot map its shard group");
        if (m->R > 1 && !m->hsdp_p2p) fail(FSDP_ERR_UNAVAILABLE, "host-collective HSDP mesh: a rank cannot map the world");
        if (m->p2p_ok) m->algo = FSDP_ALGO_P2P;
        m->hsdp_rs_p2p = m->hsdp_p2p;
      } else if (!local) {
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

fsdp_status_t fsdp_mesh_init_hostcoll(int32_t world_size, int32_t rank, int32_t shard_size, int32_t cuda_device,
                                      fsdp_host_allgather_fn fn, void* ctx, fsdp_mesh_t** out) {
  if (!fn) {
    g_last_error = "the host all-gather callback is NULL";
    return FSDP_ERR_INVALID_ARGUMENT;
  }
  if (shard_size < 0) {
    g_last_error = "shard_size must be >= 0";
    return FSDP_ERR_INVALID_ARGUMENT;
  }
  return mesh_init_impl(nullptr, world_size, rank, cuda_device, false, out, shard_size, fn, ctx);
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

fsdp_status_t fsdp_mesh_get_hsdp_rs(const fsdp_mesh_t* m, int32_t* world_pull) {
  return guarded([&] {
    if (!m || !world_pull) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    *world_pull = m->hsdp_rs_p2p ? (m->hsdp_two_phase ? 2 : 1) : 0;
  });
}

fsdp_status_t fsdp_mesh_destroy(fsdp_mesh_t* m) {
  return guarded([&] {
    if (!m) return;
    if (!m->layers.empty()) fail(FSDP_ERR_STATE, "destroy all layers of the mesh first");
    DeviceGuard g(m->device);
    for (cudaStream_t s : {m->s_cin, m->s_ag, m->s_cout, m->s_rsc, m->s_rs, m->s_ce})
      if (s) cudaStreamSynchronize(s);
    if (!m->aborted) {
      p2p_teardown(m);
    } else {   // rank-local release, no collective step
      for (auto* pool : {&m->p2p_ag, &m->p2p_rs}) {
        for (SymSlot* s : *pool) {
          sym_free_local(m, s->buf);
          if (s->free_ev) cudaEventDestroy(s->free_ev);
          if (s->cap_ev) cudaEventDestroy(s->cap_ev);
          delete s;
        }
        pool->clear();
      }
      sym_free_local(m, m->flags);
      for (SymSlot* s : m->p2p_wrs) {
        sym_free_local(m, s->buf);
        if (s->free_ev) cudaEventDestroy(s->free_ev);
        if (s->cap_ev) cudaEventDestroy(s->cap_ev);
        delete s;
      }
      m->p2p_wrs.clear();
      sym_free_local(m, m->wflags);
    }
    for (auto* pool : {&m->ag_slots, &m->rs_slots})
      for (Slot* s : *pool) {
        s->a.release(); s->b.release();
        if (s->free_ev) cudaEventDestroy(s->free_ev);
        if (s->cap_ev) cudaEventDestroy(s->cap_ev);
        delete s;
      }
    clear_presets(m);
    for (auto& r : m->prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : m->ev_pool) cudaEventDestroy(e);
    cudaFree(m->reg_acc); cudaFree(m->reg_amax); cudaFree(m->reg_scale); cudaFree(m->reg_elig);
    cudaFree(m->reg_hist); cudaFree(m->reg_pos); cudaFree(m->reg_hinit);
    if (m->h_err) cudaFreeHost(const_cast<int*>(m->h_err));
    cudaFree(m->d_barrier);
    cudaFree(m->d_epochs);
    cudaFree(m->d_wepochs);
    if (m->ev_ce) cudaEventDestroy(m->ev_ce);
    if (m->ev_pre_call) cudaEventDestroy(m->ev_pre_call);
    if (m->ev_pre_done) cudaEventDestroy(m->ev_pre_done);
    if (m->comm_rs) { if (m->aborted) ncclCommAbort(m->comm_rs); else ncclCommDestroy(m->comm_rs); }
    if (m->comm_ag) { if (m->aborted) ncclCommAbort(m->comm_ag); else ncclCommDestroy(m->comm_ag); }
    for (ncclComm_t c : {m->comm_rep, m->comm_world})
      if (c) { if (m->aborted) ncclCommAbort(c); else ncclCommDestroy(c); }
    for (cudaStream_t s : {m->s_cin, m->s_ag, m->s_cout, m->s_rsc, m->s_rs, m->s_ce})
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

fsdp_status_t fsdp_mesh_memory(const fsdp_mesh_t* m, int64_t out[4]) {
  return guarded([&] {
    if (!m || !out) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    int64_t sym = 0, pool = 0, layer = 0, peer = 0;
    auto add_sym = [&](const SymBuf& b) {   // local bytes + the group's W-1 peer mappings
      sym += (int64_t)b.bytes;
      peer += (int64_t)b.bytes * std::max<int64_t>((int64_t)b.peers.size() - 1, 0);
    };
    if (m->p2p_ok) add_sym(m->flags);
    if (m->hsdp_p2p) add_sym(m->wflags);
    for (const auto* pl : {&m->p2p_ag, &m->p2p_rs, &m->p2p_wrs})
      for (const SymSlot* s : *pl) add_sym(s->buf);
    for (const auto* pl : {&m->ag_slots, &m->rs_slots})
      for (const Slot* s : *pl) pool += (int64_t)(s->a.cap + s->b.cap);
    for (const fsdp_layer* l : m->layers) {
      layer += 2 * (int64_t)sizeof(float) * std::max<int64_t>(l->L.S, 16);   // fp32 shard + sharded grad
      if (l->gbuf) {
        if (l->gbuf_sym) add_sym(l->gbuf->buf);
        else layer += (int64_t)l->gbuf->buf.bytes;
      }
    }
    out[0] = sym;                                       // symmetric buffers this rank allocated
    out[1] = peer;                                      // the same buffers of the group's peers, mapped
    out[2] = pool;                                      // NCCL-mode / W=1 pooled buffers
    out[3] = layer;                                     // per-layer fp32 shard + grad (+ plain grad buffers)
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
    if (algo == FSDP_ALGO_NCCL && m->hc_fn) fail(FSDP_ERR_UNAVAILABLE, "a host-collective mesh has no NCCL communicator");
    for (auto* l : m->layers)
      if (l->state != SHARDED || l->rs_pending) fail(FSDP_ERR_STATE, "a layer is unsharded or has a pending reduce-scatter");
    if (algo == FSDP_ALGO_P2P && !m->p2p_ok && !m->hsdp_p2p)
      fail(FSDP_ERR_UNAVAILABLE, "P2P needs 2 <= W <= 8 ranks whose GPUs can map each other's memory");
    if (algo == FSDP_ALGO_NCCL || m->p2p_ok) m->algo = algo;   // W = 1 HSDP: the unshard stays local
    m->hsdp_rs_p2p = algo == FSDP_ALGO_P2P && m->hsdp_p2p;
  });
}

fsdp_status_t fsdp_mesh_get_algo(const fsdp_mesh_t* m, int32_t* algo) {
  return guarded([&] {
    if (!m || !algo) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    *algo = m->algo;
  });
}

fsdp_status_t fsdp_mesh_set_p2p_rs(fsdp_mesh_t* m, int32_t mode) {
  return guarded([&] {
    check_mesh(m);
    if (mode != FSDP_P2P_RS_PULL && mode != FSDP_P2P_RS_STORE && mode != FSDP_P2P_RS_AUTO)
      fail(FSDP_ERR_INVALID_ARGUMENT, "unknown P2P reduce-scatter mode");
    for (auto* l : m->layers)
      if (l->rs_pending) fail(FSDP_ERR_STATE, "a layer has a pending reduce-scatter");
    m->p2p_rs_mode = mode;
  });
}

fsdp_status_t fsdp_mesh_get_p2p_rs(const fsdp_mesh_t* m, int32_t* mode) {
  return guarded([&] {
    if (!m || !mode) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    *mode = m->p2p_rs_mode;
  });
}

fsdp_status_t fsdp_mesh_synchronize(fsdp_mesh_t* m, int64_t timeout_ms) {
  return guarded([&] {
    check_mesh(m);
    DeviceGuard g(m->device);
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t ss[] = {m->s_cin, m->s_ag, m->s_cout, m->s_rsc, m->s_rs, m->s_ce};
    for (;;) {
      bool idle = true;
      for (cudaStream_t s : ss) {
        cudaError_t e = cudaStreamQuery(s);
        if (e == cudaErrorNotReady) { idle = false; continue; }
        if (e != cudaSuccess) fail(FSDP_ERR_CUDA, std::string("stream error: ") + cudaGetErrorString(e));
      }
      if (nccl_ok(m)) {
        for (ncclComm_t c : {m->comm_ag, m->comm_rs}) {
          ncclResult_t ar = ncclSuccess;
          if (!c) continue;
          NCCL_CHECK(ncclCommGetAsyncError(c, &ar));
          if (ar != ncclSuccess) abort_mesh(m, FSDP_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(ar));
        }
      }
      if (idle) break;
      if (timeout_ms > 0 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms)) {
        if (m->comm_ag) ncclCommAbort(m->comm_ag);
        if (m->comm_rs) ncclCommAbort(m->comm_rs);
        m->comm_ag = m->comm_rs = nullptr;
        abort_mesh(m, FSDP_ERR_TIMEOUT, "mesh streams did not drain before the timeout; communicators aborted");
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    const int err = *m->h_err;
    if (err) {
      *m->h_err = 0;
      if ((err & 0xFF) == 2)   // a P2P handshake gave up waiting for a peer
        abort_mesh(m, FSDP_ERR_TIMEOUT, "P2P handshake timed out waiting for shard rank " + std::to_string(err >> 8) +
                                            " (a rank skipped or diverged from the collective call sequence); mesh aborted");
      fail(FSDP_ERR_NONFINITE, "non-finite fp8 amax seen by fsdp_precompute_fp8_scales (SPEC.md:38)");
    }
  });
}

fsdp_status_t fsdp_mesh_set_allocator(fsdp_mesh_t* m, fsdp_alloc_fn alloc_fn, fsdp_free_fn free_fn, void* ctx) {
  return guarded([&] {
    check_mesh(m);
    if ((alloc_fn == nullptr) != (free_fn == nullptr))
      fail(FSDP_ERR_INVALID_ARGUMENT, "alloc_fn and free_fn must both be set or both be NULL");
    m->allocator = Allocator{alloc_fn, free_fn, alloc_fn ? ctx : nullptr, m->device};
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

}  // extern "C"
