// C ABI, part 3: one-kernel stage entry points (all kernels testable at any W on one GPU).
#include "capi_internal.h"

using namespace fsdpc;

extern "C" {

// ------------------------------------------------------------------------- stage entry points
fsdp_status_t fsdp_stage_copy_in(const fsdp_layer_t* lc, fsdp_dtype_t dt, const float* scales, void* slot,
                                 float* amax_accum, void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    if (!slot) fail(FSDP_ERR_INVALID_ARGUMENT, "ag_slot is NULL");
    if (dt != FSDP_BFLOAT16 && dt != FSDP_FLOAT8_E4M3FN) fail(FSDP_ERR_DTYPE, "param_dtype must be BFLOAT16 or FLOAT8_E4M3FN");
    const bool fp8 = dt == FSDP_FLOAT8_E4M3FN;
    if (fp8 && !scales) scales = l->mesh->reg_scale + l->reg_base;
    DeviceGuard g(l->mesh->device);
    do_copy_in(l, fp8, scales, slot, as_stream(stream), fp8 ? reinterpret_cast<uint32_t*>(amax_accum) : nullptr);
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
    if (!l->t_amax_stage.d) {   // built once per layer (registry index = local param index)
      std::vector<Tile> tiles;
      fsdpl::append_tiles_amax(l->L, l->shard, 0, &tiles);
      if (tiles.empty()) {
        CUDA_CHECK(cudaMemsetAsync(amax_out, 0, sizeof(float) * l->P, st));
        return;
      }
      l->t_amax_stage.upload(tiles);
    }
    CUDA_CHECK(cudaMemsetAsync(amax_out, 0, sizeof(float) * l->P, st));
    CUDA_CHECK(fsdpk::launch_amax(l->t_amax_stage.d, l->t_amax_stage.n, reinterpret_cast<uint32_t*>(amax_out),
                                  l->mesh->cfg, st));
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
                                      void* const* arenas, float* amax_accum, void* stream) {
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
      check_align16(arenas[r], "arenas[r]");
      pp.p[r] = (uint8_t*)arenas[r];
    }
    DeviceGuard g(m->device);
    const DevTiles& T = fp8 ? l->t_push_fp8 : l->t_push_bf16;
    ProfScope ps(m, FSDP_PROF_UNSHARD_PUSH, as_stream(stream), fp8 ? l->push_bytes_fp8 : l->push_bytes_bf16);
    uint32_t* acc = fp8 ? reinterpret_cast<uint32_t*>(amax_accum) : nullptr;
    if (m->ce)
      ce_unshard(l, fp8, scales, pp, as_stream(stream), acc);
    else
      CUDA_CHECK(fsdpp::launch_unshard_push(T.d, T.n, l->shard, scales, pp, m->W, m->rank, m->cfg, as_stream(stream),
                                            acc));
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
      check_align16(stagings[r], "stagings[r]");
      pp.p[r] = (uint8_t*)stagings[r];
    }
    DeviceGuard g(m->device);
    ProfScope ps(m, FSDP_PROF_RS_PULL, as_stream(stream), (int64_t)(m->W - 1) * l->pull_elems * dtype_size(gd));
    CUDA_CHECK(fsdpp::launch_rs_pull(l->t_pull.d, l->t_pull.n, pp, gd == FSDP_BFLOAT16, m->W * m->R, l->grad, mean != 0,
                                     accumulate != 0, rd == FSDP_BFLOAT16, m->W, m->cfg, as_stream(stream)));
    ps.done();
  });
}

static void check_hsdp_stage(const fsdp_layer* l, int32_t replicate) {
  const fsdp_mesh* m = l->mesh;
  if (replicate < 1) fail(FSDP_ERR_INVALID_ARGUMENT, "replicate must be >= 1");
  if (m->R != 1 && m->R != replicate) fail(FSDP_ERR_INVALID_ARGUMENT, "replicate differs from the mesh's replicate size");
  if (m->W * replicate > 8) fail(FSDP_ERR_UNAVAILABLE, "the world pull supports replicate * W <= 8");
}

fsdp_status_t fsdp_stage_rs_pull_hsdp(fsdp_layer_t* l, const void* const* stagings, int32_t replicate, fsdp_dtype_t gd,
                                      fsdp_dtype_t rd, int32_t mean, int32_t accumulate, void* stream) {
  return guarded([&] {
    check_layer(l);
    check_hsdp_stage(l, replicate);
    fsdp_mesh* m = l->mesh;
    const int Wt = m->W * replicate;
    if (!stagings) fail(FSDP_ERR_INVALID_ARGUMENT, "stagings is NULL");
    if (gd != FSDP_BFLOAT16 && gd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "grad_dtype must be BFLOAT16 or FLOAT32");
    if (rd != FSDP_BFLOAT16 && rd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "reduce_dtype must be FLOAT32 or BFLOAT16");
    fsdpp::PeerPtrs pp{};
    for (int r = 0; r < Wt; ++r) {
      if (!stagings[r]) fail(FSDP_ERR_INVALID_ARGUMENT, "stagings[g] is NULL");
      check_align16(stagings[r], "stagings[g]");
      pp.p[r] = (uint8_t*)stagings[r];
    }
    DeviceGuard g(m->device);
    ProfScope ps(m, FSDP_PROF_RS_PULL, as_stream(stream), (int64_t)(Wt - 1) * l->pull_elems * dtype_size(gd));
    CUDA_CHECK(fsdpp::launch_rs_pull_nested(l->t_pull.d, l->t_pull.n, pp, gd == FSDP_BFLOAT16, Wt, l->grad, mean != 0,
                                            accumulate != 0, rd == FSDP_BFLOAT16, Wt, m->W, m->cfg, as_stream(stream)));
    ps.done();
  });
}

fsdp_status_t fsdp_stage_hsdp_piece_pull(fsdp_layer_t* l, const void* const* stagings, int32_t replicate,
                                         int32_t replica, fsdp_dtype_t gd, fsdp_dtype_t rd, int32_t mean, float* res_dev,
                                         void* stream) {
  return guarded([&] {
    check_layer(l);
    check_hsdp_stage(l, replicate);
    fsdp_mesh* m = l->mesh;
    const int Wt = m->W * replicate;
    if (replica < 0 || replica >= replicate) fail(FSDP_ERR_INVALID_ARGUMENT, "replica out of range");
    if (!stagings || !res_dev) fail(FSDP_ERR_INVALID_ARGUMENT, "NULL argument");
    check_align16(res_dev, "res_dev");
    if (gd != FSDP_BFLOAT16 && gd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "grad_dtype must be BFLOAT16 or FLOAT32");
    if (rd != FSDP_BFLOAT16 && rd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "reduce_dtype must be FLOAT32 or BFLOAT16");
    fsdpp::PeerPtrs pp{};
    for (int r = 0; r < Wt; ++r) {
      if (!stagings[r]) fail(FSDP_ERR_INVALID_ARGUMENT, "stagings[g] is NULL");
      check_align16(stagings[r], "stagings[g]");
      pp.p[r] = (uint8_t*)stagings[r];
    }
    DeviceGuard g(m->device);
    ensure_pieces(l, replicate);
    const DevTiles& T = l->t_piece[replica];
    ProfScope ps(m, FSDP_PROF_RS_PULL, as_stream(stream), (int64_t)(Wt - 1) * l->pull_elems * dtype_size(gd) / replicate);
    CUDA_CHECK(fsdpp::launch_rs_pull_nested(T.d, T.n, pp, gd == FSDP_BFLOAT16, Wt, res_dev, mean != 0, false,
                                            rd == FSDP_BFLOAT16, Wt, m->W, m->cfg, as_stream(stream)));
    ps.done();
  });
}

fsdp_status_t fsdp_stage_hsdp_replica_gather(fsdp_layer_t* l, const float* const* res_devs, int32_t replicate,
                                             int32_t accumulate, void* stream) {
  return guarded([&] {
    check_layer(l);
    check_hsdp_stage(l, replicate);
    fsdp_mesh* m = l->mesh;
    if (!res_devs) fail(FSDP_ERR_INVALID_ARGUMENT, "res_devs is NULL");
    fsdpp::PeerPtrs rp{};
    for (int q = 0; q < replicate; ++q) {
      if (!res_devs[q]) fail(FSDP_ERR_INVALID_ARGUMENT, "res_devs[q] is NULL");
      check_align16(res_devs[q], "res_devs[q]");
      rp.p[q] = (uint8_t*)res_devs[q];
    }
    DeviceGuard g(m->device);
    ensure_pieces(l, replicate);
    ProfScope ps(m, FSDP_PROF_REPLICA_GATHER, as_stream(stream), (int64_t)(replicate - 1) * 4 * l->pull_elems / replicate);
    CUDA_CHECK(fsdpp::launch_replica_gather(l->t_gather.d, l->t_gather.n, rp, l->grad, accumulate != 0, m->cfg,
                                            as_stream(stream)));
    ps.done();
  });
}

fsdp_status_t fsdp_stage_rs_scatter(const fsdp_layer_t* lc, const void* const* grads, fsdp_dtype_t gd,
                                    void* const* recv, int32_t include_self, void* stream) {
  return guarded([&] {
    fsdp_layer* l = const_cast<fsdp_layer*>(lc);
    check_layer(l);
    fsdp_mesh* m = l->mesh;
    if (m->W > 8) fail(FSDP_ERR_UNAVAILABLE, "the store-based reduce-scatter supports W <= 8");
    validate_grads(l, grads, gd, FSDP_FLOAT32);
    if (!recv) fail(FSDP_ERR_INVALID_ARGUMENT, "recv_dev is NULL");
    fsdpp::PeerPtrs pp{};
    for (int r = 0; r < m->W; ++r) {
      if (!recv[r]) fail(FSDP_ERR_INVALID_ARGUMENT, "recv_dev[r] is NULL");
      pp.p[r] = (uint8_t*)recv[r];
    }
    fsdpk::PtrArray pa{};
    for (int p = 0; p < l->P; ++p) pa.p[p] = grads[p];
    const DevTiles& T = include_self ? (gd == FSDP_BFLOAT16 ? l->t_scatter_bf16 : l->t_scatter_fp32)
                                     : (gd == FSDP_BFLOAT16 ? l->t_scatter_peers_bf16 : l->t_scatter_peers_fp32);
    DeviceGuard g(m->device);
    ProfScope ps(m, FSDP_PROF_RS_SCATTER, as_stream(stream), l->scatter_elems * dtype_size(gd));
    if (m->ce)
      ce_scatter(l, grads, dtype_size(gd), pp, as_stream(stream), include_self != 0);
    else
      CUDA_CHECK(fsdpp::launch_rs_scatter(T.d, T.n, pa, pp, m->cfg, as_stream(stream)));
    ps.done();
  });
}

fsdp_status_t fsdp_stage_rs_recv_reduce(fsdp_layer_t* l, const void* recv, const void* const* own_grads,
                                        fsdp_dtype_t gd, fsdp_dtype_t rd, int32_t mean, int32_t accumulate,
                                        void* stream) {
  return guarded([&] {
    check_layer(l);
    fsdp_mesh* m = l->mesh;
    if (m->W > 8) fail(FSDP_ERR_UNAVAILABLE, "the store-based reduce-scatter supports W <= 8");
    if (!recv) fail(FSDP_ERR_INVALID_ARGUMENT, "recv_dev is NULL");
    check_align16(recv, "recv_dev");
    if (gd != FSDP_BFLOAT16 && gd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "grad_dtype must be BFLOAT16 or FLOAT32");
    if (rd != FSDP_BFLOAT16 && rd != FSDP_FLOAT32) fail(FSDP_ERR_DTYPE, "reduce_dtype must be FLOAT32 or BFLOAT16");
    const int64_t gsz = dtype_size(gd);
    fsdpp::PeerPtrs slots{};
    for (int q = 0; q < m->W; ++q) slots.p[q] = (uint8_t*)recv + (size_t)q * l->L.S * gsz;
    fsdpk::PtrArray pa{};
    if (own_grads) {
      validate_grads(l, own_grads, gd, FSDP_FLOAT32);
      if (!(gd == FSDP_BFLOAT16 ? l->own_ok_bf16 : l->own_ok_fp32))
        fail(FSDP_ERR_INVALID_ARGUMENT, "own-row offsets of this layout are not 16-byte aligned for this grad dtype");
      for (int p = 0; p < l->P; ++p) {
        if (l->L.metas[p].row_count > 0) check_align16(own_grads[p], "own_grads_dev[p]");
        pa.p[p] = own_grads[p];
      }
    }
    DeviceGuard g(m->device);
    ProfScope ps(m, FSDP_PROF_RS_REDUCE, as_stream(stream), l->pull_elems * (m->W * gsz + 4));
    if (own_grads)
      CUDA_CHECK(fsdpp::launch_rs_reduce_own(l->t_recv_own.d, l->t_recv_own.n, recv, l->L.S, gd == FSDP_BFLOAT16, pa,
                                             l->L.rank, m->W * m->R, l->grad, mean != 0, accumulate != 0,
                                             rd == FSDP_BFLOAT16, m->W, m->cfg, as_stream(stream)));
    else
      CUDA_CHECK(fsdpp::launch_rs_pull(l->t_recv.d, l->t_recv.n, slots, gd == FSDP_BFLOAT16, m->W * m->R, l->grad,
                                       mean != 0, accumulate != 0, rd == FSDP_BFLOAT16, m->W, m->cfg, as_stream(stream)));
    ps.done();
  });
}

}  // extern "C"
