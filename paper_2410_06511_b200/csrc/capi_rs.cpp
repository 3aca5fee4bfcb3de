// C ABI reduce-scatter mechanisms (post-backward): the entry point
// fsdp_reduce_scatter_grads (capi_layer.cpp) validates the call and picks one of these —
// the HSDP world reduce-scatter on one NVSwitch domain, the P2P store or pull mechanism, or
// the NCCL path (copy-in kernel -> ncclReduceScatter -> copy-out).  Each enqueues its work on
// the mesh's streams, records l->ev_rs_done and marks the reduce-scatter pending.
#include "capi_internal.h"

namespace fsdpc {

void RsCall::replica_all_reduce(float* buf, cudaStream_t st) const {
  ProfScope pa(m, FSDP_PROF_ALL_REDUCE, st, (int64_t)2 * (m->R - 1) * S * 4 / m->R);
  NCCL_CHECK(ncclAllReduce(buf, buf, (size_t)S, ncclFloat32, ncclSum, m->comm_rep, st));
  pa.done();
}

void RsCall::add_temp_into_grad(const float* T, cudaStream_t st) const {
  ProfScope po(m, FSDP_PROF_RS_COPY_OUT, st, S * 12);
  CUDA_CHECK(fsdpk::launch_rs_copy_out(T, false, l->grad, true, S, m->cfg, st));
  po.done();
}

// HSDP on one NVSwitch domain: the (two-phase) world reduce-scatter.
void rs_hsdp_world(const RsCall& c) {
  fsdp_layer* l = c.l;
  fsdp_mesh* m = c.m;
  [[maybe_unused]] const void* const* grads = c.grads;
  [[maybe_unused]] const fsdp_dtype_t gd = c.gd;
  [[maybe_unused]] const bool obf = c.obf;
  [[maybe_unused]] const int64_t osz = c.osz, S = c.S;
  [[maybe_unused]] const bool hsdp = c.hsdp, via_temp = c.via_temp;
  [[maybe_unused]] const int divisor = c.divisor;
  [[maybe_unused]] const int32_t mean = c.mean, accumulate = c.accumulate;
  [[maybe_unused]] cudaStream_t cs = c.cs;
  [[maybe_unused]] const Capture& cap = c.cap;
  // HSDP on one NVSwitch domain (header: fsdp_mesh_init_hsdp): ONE pull over the
  // world.  Every rank stages its full grads (zero copy when they live in the layer's
  // world-symmetric grad buffer); after the world ready handshake this rank reads its
  // shard rows from all R x W ranks, divides each by R W and sums them shard ranks first,
  // then replicas (global rank order, R15) into its fp32 grad — the shard-group
  // reduce-scatter and the replica all-reduce in one kernel, bit-exact to HsdpWorld
  // 'order'.  Accumulation is the kernel's (g + sum), as the NCCL pair's temp + add.
  // Two-phase (default): replica q computes only piece q (1/R) of its shard rank's world
  // sum into the fp32 result region of its world buffer, and after the done handshake
  // every rank copies the R pieces from the R replicas of its shard rank into its grad:
  // (RW-1) 2 S / R + (R-1) 4 S / R bytes in per rank instead of (RW-1) 2 S, same bits.
  const Group G = group_of(m, GRP_WORLD);
  const int64_t gsz = dtype_size(gd);
  const int64_t res_off = hsdp_res_offset(l, gsz);
  const size_t need2 = (size_t)(res_off + 4 * std::max<int64_t>(l->L.S, 16));
  const bool use_gbuf = l->gbuf && l->gbuf_sym && l->gbuf->buf.grp == GRP_WORLD && gd == l->gbuf_dtype;
  // rank-consistent: the environment, and buffer sizes that are equal on every rank
  const bool two_phase = m->hsdp_two_phase && (!use_gbuf || l->gbuf->buf.bytes >= need2);
  bool zc = use_gbuf;
  for (int p = 0; zc && p < l->P; ++p)
    zc = l->L.numel[p] == 0 || grads[p] == (const void*)((uint8_t*)l->gbuf->buf.local + l->stg_off_el[p] * gsz);
  SymSlot* ss = use_gbuf ? l->gbuf
                         : acquire_sym_slot(m, m->p2p_wrs, two_phase ? need2 : (size_t)(l->stg_elems * gsz),
                                            (int)(m->rs_rr++ % 2), cap, GRP_WORLD);
  if (two_phase) ensure_pieces(l, m->R);
  CUDA_CHECK(cudaEventRecord(l->ev_rcall, cs));
  if (zc) {
    CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, l->ev_rcall, 0));
    wait_released(m->s_rs, ss, cap);   // the previous gather out of this buffer (s_rsc)
  } else {
    CUDA_CHECK(cudaStreamWaitEvent(m->s_rsc, l->ev_rcall, 0));
    wait_released(m->s_rsc, ss, cap);
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
  {
    ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_rs, 0);
    CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_READY, ss->index, GRP_WORLD),
                                         flag_local(m, FK_RS_READY, ss->index, GRP_WORLD), G.W, G.rank,
                                         epoch_ctr(m, FK_RS_READY, ss->index, GRP_WORLD), m->p2p_timeout_ns,
                                         m->d_err, m->s_rs, false, /*fence: staged / zero-copy grads*/ true));
    ph.done();
  }
  {
    ProfScope pp(m, FSDP_PROF_RS_PULL, m->s_rs, (int64_t)(G.W - 1) * l->pull_elems * gsz / (two_phase ? m->R : 1));
    fsdpk::LaunchCfg pcfg = m->cfg;
    if (!zc) pcfg.variant &= ~2;   // bulk pull only without a concurrent staging copy (profiles/r06)
    if (two_phase) {
      const DevTiles& T = l->t_piece[m->rep];
      CUDA_CHECK(fsdpp::launch_rs_pull_nested(T.d, T.n, peer_ptrs(m, ss->buf), gd == FSDP_BFLOAT16, divisor,
                                              (float*)((uint8_t*)ss->buf.local + res_off), mean != 0, false, obf,
                                              G.W, m->W, pcfg, m->s_rs));
    } else {
      CUDA_CHECK(fsdpp::launch_rs_pull_nested(l->t_pull.d, l->t_pull.n, peer_ptrs(m, ss->buf), gd == FSDP_BFLOAT16,
                                              divisor, l->grad, mean != 0, accumulate != 0, obf, G.W, m->W, pcfg,
                                              m->s_rs));
    }
    pp.done();
  }
  {
    ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_rs, 0);
    CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_DONE, ss->index, GRP_WORLD),
                                         flag_local(m, FK_RS_DONE, ss->index, GRP_WORLD), G.W, G.rank,
                                         epoch_ctr(m, FK_RS_DONE, ss->index, GRP_WORLD), m->p2p_timeout_ns,
                                         m->d_err, m->s_rs, m->cfg.pdl, /*fence: result pieces*/ two_phase));
    ph.done();
  }
  cudaStream_t fin = m->s_rs;
  if (two_phase) {   // every piece is final on its replica (done handshake): gather them
    // on the second stream, so the next unit's phase 1 (s_rs) overlaps this gather
    fin = m->s_rsc;
    CUDA_CHECK(cudaEventRecord(l->ev_k5, m->s_rs));
    CUDA_CHECK(cudaStreamWaitEvent(fin, l->ev_k5, 0));
    fsdpp::PeerPtrs rp{};
    for (int q = 0; q < m->R; ++q) rp.p[q] = (uint8_t*)ss->buf.peers[q * m->W + m->rank] + res_off;
    // it overlaps the next unit's phase 1 and all-gather: a smaller grid leaves them SMs
    // (FSDP_B200_GATHER_CTAS_PER_SM; 0 = the default grid)
    fsdpk::LaunchCfg gcfg = m->cfg;
    if (m->gather_per_sm > 0) gcfg.per_sm = m->gather_per_sm;
    ProfScope pg(m, FSDP_PROF_REPLICA_GATHER, fin, (int64_t)(m->R - 1) * 4 * l->pull_elems / m->R);
    CUDA_CHECK(fsdpp::launch_replica_gather(l->t_gather.d, l->t_gather.n, rp, l->grad, accumulate != 0, gcfg,
                                            fin));
    pg.done();
  }
  // the slot (staging + result pieces) is rewritten only after the next ready handshake
  // of this slot, which every rank signals after its own gather has read the pieces (the
  // zero-copy path waits for this release before that handshake)
  release_sym_slot(ss, fin, cap);
  CUDA_CHECK(cudaEventRecord(l->ev_rs_done, fin));
  l->rs_pending = true;

}

// P2P store mechanism: scatter of this rank's rows into the owners' receive buffers, local reduce.
void rs_p2p_store(const RsCall& c) {
  fsdp_layer* l = c.l;
  fsdp_mesh* m = c.m;
  [[maybe_unused]] const void* const* grads = c.grads;
  [[maybe_unused]] const fsdp_dtype_t gd = c.gd;
  [[maybe_unused]] const bool obf = c.obf;
  [[maybe_unused]] const int64_t osz = c.osz, S = c.S;
  [[maybe_unused]] const bool hsdp = c.hsdp, via_temp = c.via_temp;
  [[maybe_unused]] const int divisor = c.divisor;
  [[maybe_unused]] const int32_t mean = c.mean, accumulate = c.accumulate;
  [[maybe_unused]] cudaStream_t cs = c.cs;
  [[maybe_unused]] const Capture& cap = c.cap;
  // store-based path: ready handshake (this rank's receive buffer is free) -> scatter
  // (this rank's rows of every rank's chunk, read from the caller's grads, stored into
  // each rank's receive buffer over NVLink) -> done handshake (every rank's rows arrived)
  // on s_rs; then the local ascending-rank reduce on s_rsc, which overlaps the next
  // unit's scatter on s_rs.  The receive buffer is free again after the reduce.
  const int64_t gsz = dtype_size(gd);
  const int prefer = (int)(m->rs_rr++ % 2);
  SymSlot* ss = acquire_sym_slot(m, m->p2p_rs, (size_t)(m->W * S * gsz), prefer, cap);
  Slot* tmp = via_temp ? acquire_slot(m, m->rs_slots, 0, (size_t)(S * 4), 1, cap) : nullptr;
  CUDA_CHECK(cudaEventRecord(l->ev_rcall, cs));
  CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, l->ev_rcall, 0));
  wait_released(m->s_rs, ss, cap);
  {
    ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_rs, 0);
    CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_READY, ss->index), flag_local(m, FK_RS_READY, ss->index),
                                         m->W, m->rank, epoch_ctr(m, FK_RS_READY, ss->index), m->p2p_timeout_ns,
                                         m->d_err, m->s_rs));
    ph.done();
  }
  // own rows: read by the local reduce straight from the caller's grads (no own-slot copy,
  // 4 B of HBM per own bf16 element less) when every own-row source is 16-byte aligned;
  // purely local, so ranks may decide differently
  fsdpk::PtrArray pa{};
  for (int p = 0; p < l->P; ++p) pa.p[p] = grads[p];
  bool own_direct = m->store_own_direct && (gd == FSDP_BFLOAT16 ? l->own_ok_bf16 : l->own_ok_fp32);
  for (int p = 0; own_direct && p < l->P; ++p)
    if (l->L.metas[p].row_count > 0 && ((uintptr_t)grads[p] & 15u) != 0) own_direct = false;
  {
    const DevTiles& T = own_direct ? (gd == FSDP_BFLOAT16 ? l->t_scatter_peers_bf16 : l->t_scatter_peers_fp32)
                                   : (gd == FSDP_BFLOAT16 ? l->t_scatter_bf16 : l->t_scatter_fp32);
    ProfScope pp(m, FSDP_PROF_RS_SCATTER, m->s_rs, l->scatter_elems * gsz);
    if (m->ce)   // the copy engines move the rows (FSDP_B200_CE)
      ce_scatter(l, grads, gsz, peer_ptrs(m, ss->buf), m->s_rs, !own_direct);
    else
      CUDA_CHECK(fsdpp::launch_rs_scatter(T.d, T.n, pa, peer_ptrs(m, ss->buf), m->cfg, m->s_rs));
    pp.done();
  }
  {
    ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_rs, 0);
    CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_DONE, ss->index), flag_local(m, FK_RS_DONE, ss->index),
                                         m->W, m->rank, epoch_ctr(m, FK_RS_DONE, ss->index), m->p2p_timeout_ns,
                                         m->d_err, m->s_rs, m->cfg.pdl, m->ce));   // CE copies: no kernel fence
    ph.done();
  }
  CUDA_CHECK(cudaEventRecord(l->ev_k5, m->s_rs));
  CUDA_CHECK(cudaStreamWaitEvent(m->s_rsc, l->ev_k5, 0));
  float* target = l->grad;
  if (via_temp) {
    wait_released(m->s_rsc, tmp, cap);
    target = (float*)tmp->b.p;
    CUDA_CHECK(cudaMemsetAsync(target, 0, sizeof(float) * S, m->s_rsc));   // padding stays 0
  }
  {
    fsdpp::PeerPtrs slots{};
    for (int q = 0; q < m->W; ++q) slots.p[q] = (uint8_t*)ss->buf.local + (size_t)q * S * gsz;
    const bool acc = accumulate != 0 && !hsdp;
    fsdpk::LaunchCfg rcfg = m->cfg;   // the reduce overlaps the next unit's transfers: its grid
    if (m->reduce_per_sm > 0) rcfg.per_sm = m->reduce_per_sm;   // can leave them SMs
    ProfScope pr(m, FSDP_PROF_RS_REDUCE, m->s_rsc, l->pull_elems * (m->W * gsz + 4 + (acc ? 4 : 0)));
    if (own_direct)
      CUDA_CHECK(fsdpp::launch_rs_reduce_own(l->t_recv_own.d, l->t_recv_own.n, ss->buf.local, S, gd == FSDP_BFLOAT16,
                                             pa, l->L.rank, divisor, target, mean != 0, acc, obf, m->W, rcfg,
                                             m->s_rsc));
    else
      CUDA_CHECK(fsdpp::launch_rs_pull(l->t_recv.d, l->t_recv.n, slots, gd == FSDP_BFLOAT16, divisor, target,
                                       mean != 0, acc, obf, m->W, rcfg, m->s_rsc));
    pr.done();
  }
  release_sym_slot(ss, m->s_rsc, cap);
  if (hsdp) {
    c.replica_all_reduce(target, m->s_rsc);
    if (via_temp) {
      c.add_temp_into_grad(target, m->s_rsc);
      release_slot(tmp, m->s_rsc, cap);
    }
  }
  CUDA_CHECK(cudaEventRecord(l->ev_rs_done, m->s_rsc));
  l->rs_pending = true;

}

// P2P pull mechanism: every owner reads its rows from every rank's staged (or zero-copy) grads.
void rs_p2p_pull(const RsCall& c) {
  fsdp_layer* l = c.l;
  fsdp_mesh* m = c.m;
  [[maybe_unused]] const void* const* grads = c.grads;
  [[maybe_unused]] const fsdp_dtype_t gd = c.gd;
  [[maybe_unused]] const bool obf = c.obf;
  [[maybe_unused]] const int64_t osz = c.osz, S = c.S;
  [[maybe_unused]] const bool hsdp = c.hsdp, via_temp = c.via_temp;
  [[maybe_unused]] const int divisor = c.divisor;
  [[maybe_unused]] const int32_t mean = c.mean, accumulate = c.accumulate;
  [[maybe_unused]] cudaStream_t cs = c.cs;
  [[maybe_unused]] const Capture& cap = c.cap;
  // fused path: stage the caller's grads into this rank's symmetric staging -> ready
  // handshake -> pull (every rank's rows of this rank, /divisor, ascending-rank fp32 sum,
  // written into the grad buffer) -> done handshake (staging reusable)
  const int64_t gsz = dtype_size(gd);
  // zero copy: the caller's grads already live in this layer's symmetric grad buffer.
  // Which buffer peers pull from (and its flag slot) must be the same on every rank, so
  // it depends only on collective state: a layer with a symmetric grad buffer of this
  // dtype always reduce-scatters through it — grads given elsewhere are staged INTO it
  // (a rank-local copy) — and a layer without one always uses the pooled staging.
  const bool use_gbuf = l->gbuf && l->gbuf_sym && l->gbuf->buf.grp == GRP_SHARD && gd == l->gbuf_dtype;
  bool zc = use_gbuf;
  for (int p = 0; zc && p < l->P; ++p)
    zc = l->L.numel[p] == 0 || grads[p] == (const void*)((uint8_t*)l->gbuf->buf.local + l->stg_off_el[p] * gsz);
  SymSlot* ss = nullptr;
  if (use_gbuf) {
    ss = l->gbuf;
  } else {
    const int prefer = (int)(m->rs_rr++ % 2);   // deterministic round robin: copy of i+1 overlaps pull of i
    ss = acquire_sym_slot(m, m->p2p_rs, (size_t)(l->stg_elems * gsz), prefer, cap);
  }
  Slot* tmp = via_temp ? acquire_slot(m, m->rs_slots, 0, (size_t)(S * 4), 1, cap) : nullptr;
  CUDA_CHECK(cudaEventRecord(l->ev_rcall, cs));
  if (zc) {
    CUDA_CHECK(cudaStreamWaitEvent(m->s_rs, l->ev_rcall, 0));
  } else {
    CUDA_CHECK(cudaStreamWaitEvent(m->s_rsc, l->ev_rcall, 0));
    wait_released(m->s_rsc, ss, cap);
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
    wait_released(m->s_rs, tmp, cap);
    target = (float*)tmp->b.p;
    CUDA_CHECK(cudaMemsetAsync(target, 0, sizeof(float) * S, m->s_rs));   // padding stays 0
  }
  {
    ProfScope ph(m, FSDP_PROF_HANDSHAKE, m->s_rs, 0);
    CUDA_CHECK(fsdpp::launch_signal_wait(flag_remote(m, FK_RS_READY, ss->index), flag_local(m, FK_RS_READY, ss->index),
                                         m->W, m->rank, epoch_ctr(m, FK_RS_READY, ss->index), m->p2p_timeout_ns,
                                         m->d_err, m->s_rs, false, /*fence: staged / zero-copy grads*/ true));
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
                                         m->W, m->rank, epoch_ctr(m, FK_RS_DONE, ss->index), m->p2p_timeout_ns,
                                         m->d_err, m->s_rs, m->cfg.pdl));
    ph.done();
  }
  release_sym_slot(ss, m->s_rs, cap);
  if (hsdp) {
    c.replica_all_reduce(target, m->s_rs);
    if (via_temp) {
      c.add_temp_into_grad(target, m->s_rs);
      release_slot(tmp, m->s_rs, cap);
    }
  }
  CUDA_CHECK(cudaEventRecord(l->ev_rs_done, m->s_rs));
  l->rs_pending = true;

}

// NCCL path: K5 chunk-cat + fp32 cast + /W, ncclReduceScatter, copy-out (+ HSDP all-reduce).
void rs_nccl(const RsCall& c) {
  fsdp_layer* l = c.l;
  fsdp_mesh* m = c.m;
  [[maybe_unused]] const void* const* grads = c.grads;
  [[maybe_unused]] const fsdp_dtype_t gd = c.gd;
  [[maybe_unused]] const bool obf = c.obf;
  [[maybe_unused]] const int64_t osz = c.osz, S = c.S;
  [[maybe_unused]] const bool hsdp = c.hsdp, via_temp = c.via_temp;
  [[maybe_unused]] const int divisor = c.divisor;
  [[maybe_unused]] const int32_t mean = c.mean, accumulate = c.accumulate;
  [[maybe_unused]] cudaStream_t cs = c.cs;
  [[maybe_unused]] const Capture& cap = c.cap;
  // NCCL path.  fp32 without accumulation: the reduce-scatter (or, at W=1, K5 itself)
  // writes straight into the layer's grad buffer — the zero-copy "view" copy-out
  const bool direct = !obf && !accumulate;
  const bool need_in = comm_ready(m) || !direct;
  const size_t stage_b = (comm_ready(m) && !direct) ? (size_t)(S * osz) : 0;
  // HSDP + accumulate: the staging buffer b holds T (fp32 [S]) first; a bf16 reduce-scatter
  // output goes AFTER it (b + 4S bytes), never into T itself — widening bf16 -> fp32 in
  // place would overwrite bf16 inputs other threads have not read yet
  const size_t t_b = via_temp ? (size_t)(S * 4) + (obf ? stage_b : 0) : stage_b;
  Slot* slot = acquire_slot(m, m->rs_slots, need_in ? (size_t)(m->W * S * osz) : 0, t_b, 2, cap);
  CUDA_CHECK(cudaEventRecord(l->ev_rcall, cs));
  CUDA_CHECK(cudaStreamWaitEvent(m->s_rsc, l->ev_rcall, 0));
  wait_released(m->s_rsc, slot, cap);
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
    if (via_temp && obf) out = (uint8_t*)slot->b.p + (size_t)S * 4;   // behind T (see acquire above)
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
    c.replica_all_reduce(T, m->s_rs);
    c.add_temp_into_grad(T, m->s_rs);
  } else {
    if (!direct) {
      ProfScope po(m, FSDP_PROF_RS_COPY_OUT, m->s_rs, S * (osz + 4 + (accumulate ? 4 : 0)));
      CUDA_CHECK(fsdpk::launch_rs_copy_out(rs_out, obf, l->grad, accumulate != 0, S, m->cfg, m->s_rs));
      po.done();
    }
    if (hsdp) c.replica_all_reduce(l->grad, m->s_rs);
  }
  CUDA_CHECK(cudaEventRecord(l->ev_rs_done, m->s_rs));
  release_slot(slot, m->s_rs, cap);
  l->rs_pending = true;
}

}  // namespace fsdpc
