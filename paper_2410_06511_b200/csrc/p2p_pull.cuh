// Reduce-scatter pull kernels (see p2p.h), shared by p2p_kernels.cu (FSDP: the flat
// ascending-rank sum over the shard group) and hsdp_kernels.cu (HSDP on one NVSwitch
// domain: the nested sum over the whole world, shard ranks within a replica first, then the
// replicas — the order of PAPER.md:476's reduce-scatter followed by the replica all-reduce).
// Header-only templates in an anonymous namespace: every including TU instantiates its own.
#pragma once
#include <algorithm>

#include "dev_util.cuh"
#include "p2p.h"

namespace fsdpp {
namespace {

using namespace fsdpdev;
using fsdpk::Tile;

// ------------------------------------------------------------------- reduce-scatter pull
// Peer loads of the pull: aligned -> one streaming load; misaligned -> L1-allocating pair
// (see dev_util.cuh load4_peer_misaligned).
template <bool kGradBf16, bool kAligned>
__device__ __forceinline__ void pload4(const uint8_t* p, uint32_t k, float (&x)[4]) {
  if (kAligned) load4<kGradBf16, true>(p, 0, x);
  else load4_peer_misaligned<kGradBf16>(p, k, x);
}

template <bool kAligned>
__device__ __forceinline__ uint4 pload16(const uint8_t* p, uint32_t k) {
  if (kAligned) return ld_stream(p);
  return extract16(ld_l1_16(p - k), ld_l1_16(p - k + 16), k);
}

struct PullOps {
  float w, inv;
  bool pow2, mean, acc, bf16r;
  uint32_t chunk, stages;   // bulk pull: bytes per peer per chunk, pipeline stages
  __device__ __forceinline__ float div(float x) const {
    if (!mean) return x;
    return pow2 ? __fmul_rn(x, inv) : __fdiv_rn(x, w);
  }
  __device__ __forceinline__ float rb(float x) const {   // bf16 rounding (bf16 reduce)
    return bf16r ? bf16_lo(pack_bf16x2(x, 0.0f)) : x;
  }
};

// Sum of W terms in source order, in groups of G consecutive sources: p = the ascending fp32
// sum within a group, a = the ascending fp32 sum of the group partials.  G = W is the flat
// ascending-rank sum of the FSDP reduce-scatter; G < W is HSDP's shard-group
// reduce-scatter followed by the replica all-reduce (oracle HsdpWorld 'order'),
// with the sources in global-rank order (replica outer, R15).  Call with q = 0..W-1 in order
// (q is a compile-time constant after unrolling, so the branches fold away).
template <int W, int G>
__device__ __forceinline__ void nsum(float& a, float& p, int q, float y) {
  static_assert(G >= 1 && W % G == 0, "group size must divide the source count");
  if (q % G == 0) p = y;
  else p = __fadd_rn(p, y);
  if (q % G == G - 1) a = (q == G - 1) ? p : __fadd_rn(a, p);
}

template <int W, bool kGradBf16, bool kAligned, int G = W>
__device__ __forceinline__ void pull_body(const PeerPtrs& st, uint64_t sb, float* __restrict__ g, uint32_t nv,
                                          uint32_t k, PullOps ops) {
  constexpr uint32_t gs = kGradBf16 ? 2 : 4;
  constexpr int U = W <= 2 ? 4 : (W <= 4 ? 2 : 1);   // ~8-16 loads in flight per thread, no spills
  uint32_t v = threadIdx.x;
  for (; v + (U - 1) * kThreads < nv; v += U * kThreads) {
    float x[U][W][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < W; ++q)
        pload4<kGradBf16, kAligned>(st.p[q] + sb + (uint64_t)gs * 4 * (v + u * kThreads), k, x[u][q]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float a[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float pp = 0.0f;
#pragma unroll
        for (int q = 0; q < W; ++q) nsum<W, G>(a[j], pp, q, ops.rb(ops.div(x[u][q][j])));
        a[j] = ops.rb(a[j]);
      }
      float4* gp = reinterpret_cast<float4*>(g) + v + u * kThreads;
      if (ops.acc) {
        const float4 o = *gp;
        a[0] = __fadd_rn(o.x, a[0]); a[1] = __fadd_rn(o.y, a[1]); a[2] = __fadd_rn(o.z, a[2]); a[3] = __fadd_rn(o.w, a[3]);
      }
      *gp = make_float4(a[0], a[1], a[2], a[3]);
    }
  }
  for (; v < nv; v += kThreads) {
    float x[W][4];
#pragma unroll
    for (int q = 0; q < W; ++q) pload4<kGradBf16, kAligned>(st.p[q] + sb + (uint64_t)gs * 4 * v, k, x[q]);
    float a[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float pp = 0.0f;
#pragma unroll
      for (int q = 0; q < W; ++q) nsum<W, G>(a[j], pp, q, ops.rb(ops.div(x[q][j])));
      a[j] = ops.rb(a[j]);
    }
    float4* gp = reinterpret_cast<float4*>(g) + v;
    if (ops.acc) {
      const float4 o = *gp;
      a[0] = __fadd_rn(o.x, a[0]); a[1] = __fadd_rn(o.y, a[1]); a[2] = __fadd_rn(o.z, a[2]); a[3] = __fadd_rn(o.w, a[3]);
    }
    *gp = make_float4(a[0], a[1], a[2], a[3]);
  }
}

// 8 elements per thread per vector: one 16-byte load per source (bf16) — half the NVLink
// read requests of the 4-element mapping — and two 16-byte fp32 stores.
template <bool kGradBf16, bool kAligned>
__device__ __forceinline__ void load8e(const uint8_t* p, uint32_t k, float (&x)[8]) {
  if (kGradBf16) {
    const uint4 a = pload16<kAligned>(p, k);
    x[0] = bf16_lo(a.x); x[1] = bf16_hi(a.x); x[2] = bf16_lo(a.y); x[3] = bf16_hi(a.y);
    x[4] = bf16_lo(a.z); x[5] = bf16_hi(a.z); x[6] = bf16_lo(a.w); x[7] = bf16_hi(a.w);
  } else {
    const uint4 a = pload16<kAligned>(p, k), b = pload16<kAligned>(p + 16, k);
    x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y); x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
    x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y); x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
  }
}

template <int W, bool kGradBf16, bool kAligned, int G = W>
__device__ __forceinline__ void pull_body8(const PeerPtrs& st, uint64_t sb, float* __restrict__ g, uint32_t nv,
                                           uint32_t k, PullOps ops) {
  constexpr uint32_t gs = kGradBf16 ? 2 : 4;
  constexpr int U = W <= 4 ? 2 : 1;
  uint32_t v = threadIdx.x;
  for (; v + (U - 1) * kThreads < nv; v += U * kThreads) {
    float x[U][W][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < W; ++q)
        load8e<kGradBf16, kAligned>(st.p[q] + sb + (uint64_t)gs * 8 * (v + u * kThreads), k, x[u][q]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float a[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float pp = 0.0f;
#pragma unroll
        for (int q = 0; q < W; ++q) nsum<W, G>(a[j], pp, q, ops.rb(ops.div(x[u][q][j])));
        a[j] = ops.rb(a[j]);
      }
      float4* gp = reinterpret_cast<float4*>(g) + 2 * (v + u * kThreads);
      if (ops.acc) {
        const float4 o0 = gp[0], o1 = gp[1];
        a[0] = __fadd_rn(o0.x, a[0]); a[1] = __fadd_rn(o0.y, a[1]); a[2] = __fadd_rn(o0.z, a[2]); a[3] = __fadd_rn(o0.w, a[3]);
        a[4] = __fadd_rn(o1.x, a[4]); a[5] = __fadd_rn(o1.y, a[5]); a[6] = __fadd_rn(o1.z, a[6]); a[7] = __fadd_rn(o1.w, a[7]);
      }
      gp[0] = make_float4(a[0], a[1], a[2], a[3]);
      gp[1] = make_float4(a[4], a[5], a[6], a[7]);
    }
  }
  for (; v < nv; v += kThreads) {
    float x[W][8];
#pragma unroll
    for (int q = 0; q < W; ++q) load8e<kGradBf16, kAligned>(st.p[q] + sb + (uint64_t)gs * 8 * v, k, x[q]);
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float pp = 0.0f;
#pragma unroll
      for (int q = 0; q < W; ++q) nsum<W, G>(a[j], pp, q, ops.rb(ops.div(x[q][j])));
      a[j] = ops.rb(a[j]);
    }
    float4* gp = reinterpret_cast<float4*>(g) + 2 * v;
    if (ops.acc) {
      const float4 o0 = gp[0], o1 = gp[1];
      a[0] = __fadd_rn(o0.x, a[0]); a[1] = __fadd_rn(o0.y, a[1]); a[2] = __fadd_rn(o0.z, a[2]); a[3] = __fadd_rn(o0.w, a[3]);
      a[4] = __fadd_rn(o1.x, a[4]); a[5] = __fadd_rn(o1.y, a[5]); a[6] = __fadd_rn(o1.z, a[6]); a[7] = __fadd_rn(o1.w, a[7]);
    }
    gp[0] = make_float4(a[0], a[1], a[2], a[3]);
    gp[1] = make_float4(a[4], a[5], a[6], a[7]);
  }
}

template <int W, bool kGradBf16, int VEC, int G = W>
__global__ void __launch_bounds__(kThreads) k_rs_pull(const Tile* __restrict__ tiles, int ntiles, PeerPtrs st,
                                                      float* __restrict__ grad, PullOps ops) {
  constexpr uint32_t gs = kGradBf16 ? 2 : 4;
  pdl_wait();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const uint64_t sb = tl.src * gs;      // byte offset into every rank's staging
    float* g = grad + tl.dst;             // 16-byte aligned
    const uint32_t n = tl.n;
    const uint32_t nv = n / VEC;
    if (VEC == 8) {
      const uint32_t k = (uint32_t)(sb & 15u);
      if (k == 0) pull_body8<W, kGradBf16, true, G>(st, sb, g, nv, 0, ops);
      else pull_body8<W, kGradBf16, false, G>(st, sb, g, nv, k, ops);
    } else {
      const uint32_t k = (uint32_t)(sb & (kGradBf16 ? 7u : 15u));
      if (k == 0) pull_body<W, kGradBf16, true, G>(st, sb, g, nv, 0, ops);
      else pull_body<W, kGradBf16, false, G>(st, sb, g, nv, k, ops);
    }
    for (uint32_t e = nv * VEC + threadIdx.x; e < n; e += kThreads) {
      float a = 0.0f, pp = 0.0f;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const uint8_t* p = st.p[q] + sb + (uint64_t)gs * e;
        const float x = kGradBf16 ? __uint_as_float(((uint32_t)(*(const uint16_t*)p)) << 16) : *(const float*)p;
        nsum<W, G>(a, pp, q, ops.rb(ops.div(x)));
      }
      a = ops.rb(a);
      g[e] = ops.acc ? __fadd_rn(g[e], a) : a;
    }
  }
}


constexpr uint32_t kPullMaxStages = 4;
constexpr size_t kPullMaxSmem = 200 * 1024;   // stages * W * chunk, leaves room for 1 CTA/SM

// kSel (W = 1 only): each tile reads its one source st.p[tile.pad] instead of st.p[0] — the
// HSDP replica gather (fp32 pieces from the replica that finished them; mean off, W = 1, so
// the "sum" is the value itself, + the grad under accumulate).
template <int W, bool kGradBf16, int G = W, bool kSel = false>
__global__ void __launch_bounds__(kThreads) k_rs_pull_bulk(const Tile* __restrict__ tiles, int ntiles, PeerPtrs st,
                                                           float* __restrict__ grad, PullOps ops) {
  static_assert(!kSel || W == 1, "per-tile source selection is the single-source (gather) form");
  extern __shared__ __align__(128) uint8_t smem[];   // [stages][W][chunk]
  __shared__ uint64_t full[kPullMaxStages];
  constexpr uint32_t gs = kGradBf16 ? 2 : 4;
  pdl_wait();
  const uint32_t chunk = ops.chunk, NS = ops.stages;
  const uint32_t CE = chunk / gs;                      // elements per chunk
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // One chunk stream across all of this CTA's tiles: thread 0 keeps the TMA issue cursor NS
  // chunks ahead of consumption, also across tile boundaries (a per-tile prologue would expose
  // one NVLink round trip per tile).  Misaligned tiles take the register path and are skipped
  // by the issue cursor.  consumed / issued count bulk chunks: stage = i % NS, parity (i/NS)&1.
  auto bulk_ok = [&](const Tile& tl) { return ((tl.src * gs) & 15u) == 0 && ((tl.n * gs) & 15u) == 0; };
  uint32_t consumed = 0;
  uint32_t issued = 0, it_c = 0;   // thread 0 only
  int it_t = blockIdx.x;           // thread 0 only: tile of the next chunk to issue
  auto advance_issue = [&]() {
    while (issued < consumed + NS && it_t < ntiles) {
      const Tile tl = tiles[it_t];
      if (!bulk_ok(tl)) { it_t += gridDim.x; it_c = 0; continue; }
      const uint32_t nch = (tl.n + CE - 1) / CE;
      const uint32_t s = issued % NS;
      const uint32_t bytes = min(CE, tl.n - it_c * CE) * gs;
      const uint64_t off = tl.src * gs + (uint64_t)it_c * chunk;
      mbar_arrive_expect_tx(&full[s], W * bytes);
#pragma unroll
      for (int q = 0; q < W; ++q)
        bulk_g2s(smem + ((size_t)s * W + q) * chunk, (kSel ? st.p[tl.pad] : st.p[q]) + off, bytes, &full[s]);
      ++issued;
      if (++it_c == nch) { it_t += gridDim.x; it_c = 0; }
    }
  };
  if (threadIdx.x == 0) advance_issue();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const uint64_t sb = tl.src * gs;
    float* g = grad + tl.dst;
    const uint32_t n = tl.n;
    if (!bulk_ok(tl)) {   // bulk needs 16-byte granularity
      PeerPtrs sel{};
      if constexpr (kSel) sel.p[0] = st.p[tl.pad];
      const PeerPtrs& sp = kSel ? sel : st;
      const uint32_t k = (uint32_t)(sb & (kGradBf16 ? 7u : 15u));
      const uint32_t nv = n / 4;
      if (k == 0) pull_body<W, kGradBf16, true, G>(sp, sb, g, nv, 0, ops);
      else pull_body<W, kGradBf16, false, G>(sp, sb, g, nv, k, ops);
      for (uint32_t e = nv * 4 + threadIdx.x; e < n; e += kThreads) {
        float a = 0.0f, pp = 0.0f;
#pragma unroll
        for (int q = 0; q < W; ++q) {
          const uint8_t* p = sp.p[q] + sb + (uint64_t)gs * e;
          const float x = kGradBf16 ? __uint_as_float(((uint32_t)(*(const uint16_t*)p)) << 16) : *(const float*)p;
          nsum<W, G>(a, pp, q, ops.rb(ops.div(x)));
        }
        a = ops.rb(a);
        g[e] = ops.acc ? __fadd_rn(g[e], a) : a;
      }
      continue;
    }
    const uint32_t nch = (n + CE - 1) / CE;
    for (uint32_t c = 0; c < nch; ++c) {
      const uint32_t i = consumed, s = i % NS;
      mbar_wait(&full[s], (i / NS) & 1u);
      const uint32_t ne = min(CE, n - c * CE);
      float* gc = g + (size_t)c * CE;
      for (uint32_t e4 = threadIdx.x; e4 * 4 < ne; e4 += kThreads) {
        float a[4], pp[4];
#pragma unroll
        for (int q = 0; q < W; ++q) {
          const uint8_t* sp = smem + ((size_t)s * W + q) * chunk + (size_t)e4 * 4 * gs;
          float x[4];
          if (kGradBf16) {
            const uint2 u = *reinterpret_cast<const uint2*>(sp);
            x[0] = bf16_lo(u.x); x[1] = bf16_hi(u.x); x[2] = bf16_lo(u.y); x[3] = bf16_hi(u.y);
          } else {
            const float4 u = *reinterpret_cast<const float4*>(sp);
            x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) nsum<W, G>(a[j], pp[j], q, ops.rb(ops.div(x[j])));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = ops.rb(a[j]);
        float4* gp = reinterpret_cast<float4*>(gc) + e4;
        if (ops.acc) {
          const float4 o = *gp;
          a[0] = __fadd_rn(o.x, a[0]); a[1] = __fadd_rn(o.y, a[1]); a[2] = __fadd_rn(o.z, a[2]); a[3] = __fadd_rn(o.w, a[3]);
        }
        *gp = make_float4(a[0], a[1], a[2], a[3]);
      }
      __syncthreads();   // everyone is done with stage s before the TMA refills it
      ++consumed;
      if (threadIdx.x == 0) advance_issue();
    }
  }
}

inline int grid_for(int64_t items, fsdpk::LaunchCfg cfg, int tuned = fsdpk::kCtasCopy) {
  const int64_t cap = cfg.cap(tuned);
  int64_t g = items < cap ? items : cap;
  return (int)(g < 1 ? 1 : g);
}

// persistent launch, programmatic (the kernel starts with pdl_wait) unless disabled
template <class... KArgs, class... Args>
cudaError_t launch_p(bool pdl, void (*kern)(KArgs...), int g, size_t smem, cudaStream_t s, Args&&... args) {
  if (pdl) return launch_persistent_pdl(kern, g, smem, s, static_cast<Args&&>(args)...);
  return launch_persistent(kern, g, smem, s, static_cast<Args&&>(args)...);
}

template <bool kGradBf16, int V>
cudaError_t launch_pull_wv(const Tile* tiles, int ntiles, PeerPtrs st, float* grad, PullOps ops, int W, int g,
                           cudaStream_t s, bool pdl) {
  switch (W) {
    case 1: return launch_p(pdl, k_rs_pull<1, kGradBf16, V>, g, 0, s, tiles, ntiles, st, grad, ops);
    case 2: return launch_p(pdl, k_rs_pull<2, kGradBf16, V>, g, 0, s, tiles, ntiles, st, grad, ops);
    case 3: return launch_p(pdl, k_rs_pull<3, kGradBf16, V>, g, 0, s, tiles, ntiles, st, grad, ops);
    case 4: return launch_p(pdl, k_rs_pull<4, kGradBf16, V>, g, 0, s, tiles, ntiles, st, grad, ops);
    case 5: return launch_p(pdl, k_rs_pull<5, kGradBf16, V>, g, 0, s, tiles, ntiles, st, grad, ops);
    case 6: return launch_p(pdl, k_rs_pull<6, kGradBf16, V>, g, 0, s, tiles, ntiles, st, grad, ops);
    case 7: return launch_p(pdl, k_rs_pull<7, kGradBf16, V>, g, 0, s, tiles, ntiles, st, grad, ops);
    case 8: return launch_p(pdl, k_rs_pull<8, kGradBf16, V>, g, 0, s, tiles, ntiles, st, grad, ops);
    default: return cudaErrorInvalidValue;
  }
}

template <int W, bool kGradBf16, int G = W, bool kSel = false>
cudaError_t launch_pull_bulk_w(const Tile* tiles, int ntiles, PeerPtrs st, float* grad, PullOps ops, int g,
                               cudaStream_t s, bool pdl) {
  while ((size_t)ops.stages * W * ops.chunk > kPullMaxSmem) {   // shrink stages, then chunk
    if (ops.stages > 2) --ops.stages;
    else ops.chunk /= 2;
  }
  const size_t smem = (size_t)ops.stages * W * ops.chunk;
  static bool attr[64] = {};   // function attributes are per device: set once per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_rs_pull_bulk<W, kGradBf16, G, kSel>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kPullMaxSmem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  // one wave (launch_persistent): at W = 8 the 64 KB stages allow 3 CTAs per SM, not 4
  return launch_p(pdl, k_rs_pull_bulk<W, kGradBf16, G, kSel>, g, smem, s, tiles, ntiles, st, grad, ops);
}

template <bool kGradBf16>
cudaError_t launch_pull_w(const Tile* tiles, int ntiles, PeerPtrs st, float* grad, PullOps ops, int W, int g,
                          cudaStream_t s, int variant, bool pdl) {
  if (variant & 2) {   // TMA bulk pull
    switch (W) {
      case 1: return launch_pull_bulk_w<1, kGradBf16>(tiles, ntiles, st, grad, ops, g, s, pdl);
      case 2: return launch_pull_bulk_w<2, kGradBf16>(tiles, ntiles, st, grad, ops, g, s, pdl);
      case 3: return launch_pull_bulk_w<3, kGradBf16>(tiles, ntiles, st, grad, ops, g, s, pdl);
      case 4: return launch_pull_bulk_w<4, kGradBf16>(tiles, ntiles, st, grad, ops, g, s, pdl);
      case 5: return launch_pull_bulk_w<5, kGradBf16>(tiles, ntiles, st, grad, ops, g, s, pdl);
      case 6: return launch_pull_bulk_w<6, kGradBf16>(tiles, ntiles, st, grad, ops, g, s, pdl);
      case 7: return launch_pull_bulk_w<7, kGradBf16>(tiles, ntiles, st, grad, ops, g, s, pdl);
      case 8: return launch_pull_bulk_w<8, kGradBf16>(tiles, ntiles, st, grad, ops, g, s, pdl);
      default: return cudaErrorInvalidValue;
    }
  }
  return (variant & 1) ? launch_pull_wv<kGradBf16, 8>(tiles, ntiles, st, grad, ops, W, g, s, pdl)
                       : launch_pull_wv<kGradBf16, 4>(tiles, ntiles, st, grad, ops, W, g, s, pdl);
}

PullOps make_ops(int divisor, bool mean, bool accumulate, bool bf16_reduce, const fsdpk::LaunchCfg& cfg) {
  PullOps ops;
  ops.w = (float)divisor;
  ops.inv = 1.0f / (float)divisor;
  ops.pow2 = (divisor & (divisor - 1)) == 0;
  ops.mean = mean;
  ops.acc = accumulate;
  ops.bf16r = bf16_reduce;
  ops.chunk = (uint32_t)cfg.pull_chunk;
  ops.stages = (uint32_t)std::min<int>(std::max(cfg.pull_stages, 2), (int)kPullMaxStages);
  return ops;
}

}  // namespace
}  // namespace fsdpp
