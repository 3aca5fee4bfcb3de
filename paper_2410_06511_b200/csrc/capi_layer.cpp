// C ABI, part 2: shard, fp8 scale precompute, unshard / reshard, reduce-scatter (NCCL and
// fused P2P paths), sharded-grad accessors, zero-copy grad buffers.
#include "capi_internal.h"

using namespace fsdpc;

extern "C" {

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
      std::vector<uint64_t> h(m->W);
      group_allgather_host(m, GRP_SHARD, &L.hash, h.data(), sizeof(uint64_t));
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
      l->al = m->allocator;
      l->shard = static_cast<float*>(l->al.allocate(sbytes));
      l->grad = static_cast<float*>(l->al.allocate(sbytes));
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
      for (int f = 0; f < 2; ++f) {   // push tables are param-major: first tile of every param
        const std::vector<Tile> tp = fsdpl::tiles_push(Ly, f == 1);
        std::vector<int>& off = f ? l->push_tile_off_fp8 : l->push_tile_off_bf16;
        off.assign(n + 1, 0);
        for (const Tile& x : tp) off[x.param + 1]++;
        for (int p = 0; p < n; ++p) off[p + 1] += off[p];
        (f ? l->t_push_fp8 : l->t_push_bf16).upload(tp);
      }
      l->t_pull.upload(fsdpl::tiles_pull(Ly, l->stg_off_el));
      l->t_stage_bf16.upload(fsdpl::tiles_stage(Ly, l->stg_off_el, 2));
      l->t_stage_fp32.upload(fsdpl::tiles_stage(Ly, l->stg_off_el, 4));
      l->t_scatter_bf16.upload(fsdpl::tiles_scatter(Ly, 2));
      l->t_scatter_fp32.upload(fsdpl::tiles_scatter(Ly, 4));
      l->t_recv.upload(fsdpl::tiles_recv_reduce(Ly));
      l->t_scatter_peers_bf16.upload(fsdpl::tiles_scatter(Ly, 2, false));
      l->t_scatter_peers_fp32.upload(fsdpl::tiles_scatter(Ly, 4, false));
      l->t_recv_own.upload(fsdpl::tiles_recv_reduce_own(Ly));
      l->own_ok_bf16 = fsdpl::own_rows_aligned(Ly, 2);
      l->own_ok_fp32 = fsdpl::own_rows_aligned(Ly, 4);
      if (m->hsdp_p2p) ensure_pieces(l, m->R);   // at shard time: no upload inside a graph capture
      for (int p = 0; p < n; ++p) {
        const int64_t cnt = Ly.metas[p].row_count * Ly.metas[p].rest;
        const int64_t es8 = Ly.fp8[p] ? 1 : 2;
        l->push_bytes_bf16 += (int64_t)(m->W - 1) * cnt * 2;      // NVLink egress
        l->push_bytes_fp8 += (int64_t)(m->W - 1) * cnt * es8;
        l->local_push_bf16 += cnt * (4 + 2);                        // W=1: HBM read + write
        l->local_push_fp8 += cnt * (4 + es8);
        l->pull_elems += cnt;
        l->scatter_elems += Ly.numel[p] - cnt;                       // the other ranks' rows
      }
      l->arena_is_flat_bf16 = Ly.arena_bf16 >= 2 * Ly.S;
      for (int p = 0; p < n; ++p)
        if (Ly.uoff_bf16[p] != 2 * Ly.metas[p].elem_offset) l->arena_is_flat_bf16 = false;
      for (int p = 0; p < n; ++p) {
        const int64_t es = Ly.fp8[p] ? 1 : 2;
        l->bytes_cin_fp8 += Ly.metas[p].padded_numel * (4 + es);
        l->bytes_cout_bf16 += 2 * 2 * Ly.numel[p];
        l->bytes_cout_fp8 += 2 * es * Ly.numel[p];
        l->grad_numel_total += Ly.numel[p];
      }
      // fp8 registry entries [reg_base, reg_base + P)
      l->reg_base = registry_reserve(m, n);
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
    for (cudaStream_t s : {m->s_cin, m->s_ag, m->s_cout, m->s_rsc, m->s_rs, m->s_ce}) cudaStreamSynchronize(s);
    l->al.release(l->shard);
    l->al.release(l->grad);
    cudaFree(l->d_idx_local);
    l->t_cin_fp8.release(); l->t_cout_bf16.release(); l->t_cout_fp8.release(); l->t_rsin.release();
    l->t_push_bf16.release(); l->t_push_fp8.release(); l->t_pull.release(); l->t_stage_bf16.release();
    l->t_stage_fp32.release(); l->t_amax_stage.release();
    l->t_scatter_bf16.release(); l->t_scatter_fp32.release(); l->t_recv.release();
    l->t_scatter_peers_bf16.release(); l->t_scatter_peers_fp32.release(); l->t_recv_own.release();
    l->t_amax_reg.release();
    for (auto& t : l->t_piece) t.release();
    l->t_gather.release();
    if (l->gbuf) {
      if (l->gbuf_sym && !m->aborted) sym_free(m, l->gbuf->buf);   // collective
      else if (l->gbuf_sym) sym_free_local(m, l->gbuf->buf);
      else l->al.release(l->gbuf->buf.local);
      if (l->gbuf->free_ev) cudaEventDestroy(l->gbuf->free_ev);
      if (l->gbuf->cap_ev) cudaEventDestroy(l->gbuf->cap_ev);
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
    if (!ps && capture_of(as_stream(stream)).on)
      fail(FSDP_ERR_STATE, "first precompute of this layer list inside a CUDA graph capture: run it once eagerly first");
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
    // delayed scaling with the amax fused into the fp8 casts: when every layer was armed by a
    // previous delayed call, the accumulator already holds the max |x| the fp8 unshards since
    // then saw — that step's amax, recorded now (K1c) exactly as K1b would have recorded it
    // after use — so the K1 pass over all fp32 shards is skipped.  An armed layer that was not
    // fp8-unsharded since (nothing accumulated) gets a K1 pass of its current parameters.
    const bool delayed = history_len > 0;
    bool fused = delayed && m->amax_fuse && m->hist_len == history_len;
    for (fsdp_layer* l : key) fused = fused && l->amax_armed;
    CUDA_CHECK(cudaEventRecord(m->ev_pre_call, st));
    CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, m->ev_pre_call, 0));
    if (!fused) {
      ProfScope pa(m, FSDP_PROF_AMAX, m->s_rs, ps->bytes);
      CUDA_CHECK(fsdpk::launch_amax(ps->tiles.d, ps->tiles.n, m->reg_acc, m->cfg, m->s_rs));
      pa.done();
    } else {
      for (fsdp_layer* l : key) {
        if (l->amax_pushed) continue;
        if (!l->t_amax_reg.d) {
          std::vector<Tile> tiles;
          fsdpl::append_tiles_amax(l->L, l->shard, l->reg_base, &tiles);
          if (tiles.empty()) continue;
          if (capture_of(st).on) fail(FSDP_ERR_STATE, "first stand-in amax pass of a layer inside a CUDA graph capture");
          l->t_amax_reg.upload(tiles);
        }
        int64_t b = 0;
        for (int p = 0; p < l->P; ++p) if (l->L.fp8[p]) b += 4 * l->L.metas[p].padded_numel;
        ProfScope pa(m, FSDP_PROF_AMAX, m->s_rs, b);
        CUDA_CHECK(fsdpk::launch_amax(l->t_amax_reg.d, l->t_amax_reg.n, m->reg_acc, m->cfg, m->s_rs));
        pa.done();
      }
    }
    if (comm_ready(m) && m->reg_size > 0) {
      // max of non-negative fp32 bit patterns == uint32 max (NaN patterns propagate)
      ProfScope pr(m, FSDP_PROF_ALL_REDUCE, m->s_rs, (int64_t)4 * m->reg_size);
      if (m->p2p_ok && (m->algo == FSDP_ALGO_P2P || !nccl_ok(m)))   // through symmetric memory
        p2p_amax_allreduce(m, m->reg_size, m->s_rs);
      else
        NCCL_CHECK(ncclAllReduce(m->reg_acc, m->reg_acc, (size_t)m->reg_size, ncclUint32, ncclMax, m->comm_rs, m->s_rs));
      pr.done();
    }
    {
      ProfScope pk(m, FSDP_PROF_SCALE, m->s_rs, (int64_t)ps->nidx * 12);
      if (history_len == 0) {
        CUDA_CHECK(fsdpk::launch_fp8_scale(ps->idx, ps->nidx, m->reg_acc, m->reg_amax, m->reg_scale, m->reg_elig,
                                           m->d_err, true, m->s_rs));
      } else if (fused) {
        CUDA_CHECK(fsdpk::launch_fp8_scale_delayed_fused(ps->idx, ps->nidx, m->reg_acc, m->reg_amax, m->reg_scale,
                                                         m->reg_elig, m->reg_hist, m->reg_pos, m->reg_hinit,
                                                         history_len, kHistMax, m->d_err, m->s_rs));
      } else {
        registry_ensure_hist(m);
        m->hist_len = history_len;
        CUDA_CHECK(fsdpk::launch_fp8_scale_delayed(ps->idx, ps->nidx, m->reg_acc, m->reg_amax, m->reg_scale,
                                                   m->reg_elig, m->reg_hist, m->reg_pos, m->reg_hinit, history_len,
                                                   kHistMax, m->d_err, m->s_rs));
      }
      pk.done();
    }
    for (fsdp_layer* l : key) {   // arm (delayed + fused) or disarm the casts' accumulation
      l->amax_armed = delayed && m->amax_fuse;
      l->amax_pushed = false;
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
    // delayed scaling, amax fused into the cast: fold max |x| into the registry accumulator
    uint32_t* amax_acc = (fp8 && l->amax_armed) ? m->reg_acc + l->reg_base : nullptr;
    if (amax_acc) l->amax_pushed = true;
    DeviceGuard g(m->device);
    const int64_t sb = slot_bytes(l, fp8);
    const int64_t arena = fp8 ? l->L.arena_fp8 : l->L.arena_bf16;
    const Capture cap = capture_of(as_stream(compute));
    if (m->algo == FSDP_ALGO_P2P) {
      // fused path: ready handshake -> push (cast + store into every rank's arena) -> done
      SymSlot* ss = acquire_sym_slot(m, m->p2p_ag, (size_t)arena, -1, cap);
      cudaStream_t cs = as_stream(compute);
      CUDA_CHECK(cudaEventRecord(l->ev_call, cs));
      CUDA_CHECK(cudaStreamWaitEvent(m->s_ag, l->ev_call, 0));
      wait_released(m->s_ag, ss, cap);
      {
        ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_ag, 0);
        CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_AG_READY, ss->index), flag_local(m, FK_AG_READY, ss->index),
                                             m->W, m->rank, epoch_ctr(m, FK_AG_READY, ss->index), m->p2p_timeout_ns,
                                             m->d_err, m->s_ag));
        ph.done();
      }
      {
        const DevTiles& T = fp8 ? l->t_push_fp8 : l->t_push_bf16;
        ProfScope pp(m, FSDP_PROF_UNSHARD_PUSH, m->s_ag, fp8 ? l->push_bytes_fp8 : l->push_bytes_bf16);
        if (m->ce)   // cast locally, the copy engines send the rows (FSDP_B200_CE)
          ce_unshard(l, fp8, scales, peer_ptrs(m, ss->buf), m->s_ag, amax_acc);
        else
          CUDA_CHECK(fsdpp::launch_unshard_push(T.d, T.n, l->shard, scales, peer_ptrs(m, ss->buf), m->W, m->rank,
                                                m->cfg, m->s_ag, amax_acc));
        pp.done();
      }
      {
        ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_ag, 0);
        CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_AG_DONE, ss->index), flag_local(m, FK_AG_DONE, ss->index),
                                             m->W, m->rank, epoch_ctr(m, FK_AG_DONE, ss->index), m->p2p_timeout_ns,
                                             m->d_err, m->s_ag, m->cfg.pdl, m->ce));   // CE copies: no kernel fence
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
      Slot* slot = acquire_slot(m, m->ag_slots, 0, (size_t)arena, 1, cap);
      cudaStream_t cs = as_stream(compute);
      CUDA_CHECK(cudaEventRecord(l->ev_call, cs));
      CUDA_CHECK(cudaStreamWaitEvent(m->s_cin, l->ev_call, 0));
      wait_released(m->s_cin, slot, cap);
      fsdpp::PeerPtrs pp{};
      pp.p[0] = (uint8_t*)slot->b.p;
      const DevTiles& T = fp8 ? l->t_push_fp8 : l->t_push_bf16;
      {
        ProfScope pc(m, FSDP_PROF_COPY_IN, m->s_cin, fp8 ? l->local_push_fp8 : l->local_push_bf16);
        if (!fp8 && l->arena_is_flat_bf16 && (m->cfg.variant & 32)) {
          // opt-in (FSDP_B200_VARIANT bit 32): when the arena has the flat shard's layout (every
          // Llama layout) the unshard is one contiguous cast, K2 straight into the unsharded
          // tensors: faster alone (6138 vs 6002 GB/s) but the overlapped W=1 step is 0.2%
          // slower next to the concurrent K5 (profiles/r13), so the push stays the default
          CUDA_CHECK(fsdpk::launch_copy_in_bf16(l->shard, slot->b.p, l->L.S, m->cfg, m->s_cin));
        } else if (m->cfg.variant & 64) {
          // FSDP_B200_VARIANT bit 64 (default): the cast with TMA loads and stores, 3 stages —
          // bf16: 226 us per 8B block, 0.983 of the copy peak, vs 239 us for the push
          // (profiles/round2/r2cast); the fp8 unshard (mixed tiles, fused amax) likewise
          CUDA_CHECK(fsdpp::launch_cast_w1(T.d, T.n, l->shard, fp8 ? scales : nullptr, slot->b.p, amax_acc, m->cfg,
                                           m->s_cin));
        } else {
          fsdpk::LaunchCfg lcfg = m->cfg;   // W = 1: bulk stores too (0.915 vs 0.902 of HBM, r06)
          if (const char* e = std::getenv("FSDP_B200_W1_BULK")) if (std::atoi(e) == 0) lcfg.variant &= ~4;
          CUDA_CHECK(fsdpp::launch_unshard_push(T.d, T.n, l->shard, scales, pp, 1, 0, lcfg, m->s_cin, amax_acc));
        }
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
    Slot* slot = acquire_slot(m, m->ag_slots, (size_t)(m->W * sb), (size_t)arena, 1, cap);
    cudaStream_t cs = as_stream(compute);
    // copy-in after the caller's prior work (optimizer step on the shard) and after the
    // previous user of this buffer released it
    CUDA_CHECK(cudaEventRecord(l->ev_call, cs));
    CUDA_CHECK(cudaStreamWaitEvent(m->s_cin, l->ev_call, 0));
    wait_released(m->s_cin, slot, cap);
    uint8_t* ag = (uint8_t*)slot->a.p;
    do_copy_in(l, fp8, scales, ag + (size_t)m->rank * sb, m->s_cin, amax_acc);
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
    poll_async_errors(l->mesh);
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
    const Capture cap = capture_of(cs);
    if (l->state == UNSHARDING) CUDA_CHECK(cudaStreamWaitEvent(cs, l->ev_done, 0));
    // the buffer is free once everything enqueued on `compute` so far (the consumers of
    // the unsharded params) has run; the next user's copy-in waits on this event
    if (l->p2p_slot) {
      // peers write into this arena only after this rank's next ready handshake on it,
      // which the next unshard issues after waiting on free_ev
      release_sym_slot(l->p2p_slot, cs, cap);
      l->p2p_slot = nullptr;
    } else {
      release_slot(l->slot, cs, cap);
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
    const RsCall c{l, m, grads, gd, obf, osz, S, hsdp, divisor, via_temp, mean, accumulate, cs, capture_of(cs)};
    if (hsdp && m->hsdp_rs_p2p) return rs_hsdp_world(c);
    // P2P mechanism: identical on every rank (the mode is set collectively; the layer's
    // zero-copy buffer exists on all ranks or none)
    // AUTO: with zero-copy buffers the pull needs no staging and one kernel less, so it wins
    // at W = 2 and for small units (the store's ~5% link-rate edge is worth less than its
    // extra kernel below ~64 MB of bus bytes, profiles/r16 alpha-B fits); else store
    const bool zc_layer = l->gbuf && l->gbuf_sym && l->gbuf->buf.grp == GRP_SHARD;
    const int64_t bus_bytes = l->stg_elems * dtype_size(gd) * (m->W - 1) / std::max(m->W, 1);
    const bool p2p_store = m->p2p_rs_mode == FSDP_P2P_RS_STORE ||
                           (m->p2p_rs_mode == FSDP_P2P_RS_AUTO &&
                            (m->ce || !(zc_layer && (m->W == 2 || bus_bytes < (64ll << 20)))));
    if (m->algo == FSDP_ALGO_P2P && p2p_store) return rs_p2p_store(c);
    if (m->algo == FSDP_ALGO_P2P) return rs_p2p_pull(c);
    rs_nccl(c);
  });
}

fsdp_status_t fsdp_wait_reduce_scatter(fsdp_layer_t* l, void* compute) {
  return guarded([&] {
    check_layer(l);
    if (!l->rs_pending) return;
    poll_async_errors(l->mesh);
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
      size_t bytes = (size_t)std::max<int64_t>(l->stg_elems, 128) * gsz;
      if (m->hsdp_rs_p2p)   // + the two-phase HSDP reduce-scatter's fp32 result region [S]
        bytes = (size_t)(hsdp_res_offset(l, gsz) + 4 * std::max<int64_t>(l->L.S, 16));
      if (m->p2p_ok || m->hsdp_rs_p2p) {   // collective: every rank of the group maps every peer's buffer
        if (kPoolSlots + m->gbuf_seq >= kAmaxSlot) fail(FSDP_ERR_UNAVAILABLE, "too many layer grad buffers");
        s->index = kPoolSlots + m->gbuf_seq++;
        // HSDP world pull: the buffer is symmetric over the whole world (its reduce-scatter
        // reads it from every replica); else over the shard group
        if (!sym_alloc(m, s->buf, bytes, m->hsdp_rs_p2p ? GRP_WORLD : GRP_SHARD)) {
          cudaEventDestroy(s->free_ev);
          delete s;
          fail(FSDP_ERR_OUT_OF_MEMORY, "symmetric grad buffer allocation/mapping failed");
        }
        l->gbuf_sym = true;
      } else {
        try {
          s->buf.local = l->al.allocate(bytes + 256);
        } catch (...) {
          cudaEventDestroy(s->free_ev);
          delete s;
          throw;
        }
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

