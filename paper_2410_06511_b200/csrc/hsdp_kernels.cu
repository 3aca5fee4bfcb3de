// HSDP reduce-scatter on one NVSwitch domain (see p2p.h launch_rs_pull_nested): the pull
// kernels of p2p_pull.cuh instantiated for W = R * G world ranks summed in groups of G.
// Separate TU so the nested instances compile in parallel with p2p_kernels.cu.
#include "p2p_pull.cuh"

namespace fsdpp {
namespace {

template <bool kGradBf16, int W, int G>
cudaError_t launch_nested_wg(const Tile* tiles, int ntiles, PeerPtrs st, float* grad, PullOps ops, int g,
                             cudaStream_t s, int variant, bool pdl) {
  if (variant & 2) return launch_pull_bulk_w<W, kGradBf16, G>(tiles, ntiles, st, grad, ops, g, s, pdl);
  return launch_p(pdl, k_rs_pull<W, kGradBf16, 8, G>, g, 0, s, tiles, ntiles, st, grad, ops);
}

template <bool kGradBf16>
cudaError_t launch_nested(const Tile* tiles, int ntiles, PeerPtrs st, float* grad, PullOps ops, int W, int G, int g,
                          cudaStream_t s, int variant, bool pdl) {
#define FSDP_WG(w, gg) \
  if (W == w && G == gg) return launch_nested_wg<kGradBf16, w, gg>(tiles, ntiles, st, grad, ops, g, s, variant, pdl);
  FSDP_WG(2, 1) FSDP_WG(3, 1) FSDP_WG(4, 1) FSDP_WG(4, 2) FSDP_WG(5, 1) FSDP_WG(6, 1)
  FSDP_WG(6, 2) FSDP_WG(6, 3) FSDP_WG(7, 1) FSDP_WG(8, 1) FSDP_WG(8, 2) FSDP_WG(8, 4)
#undef FSDP_WG
  return cudaErrorInvalidValue;
}

// Phase 2 of the two-phase HSDP reduce-scatter: grad[dst + e] (+)= res.p[tile.pad][dst + e]
// — piece q of this shard rank's world sum, finished by replica q in its result buffer (peer
// memory over NVLink, or local for q = own replica).  fp32 bits are copied (or added once
// for accumulate), so the result stays the phase-1 nested sum bit for bit.  Tile dst is
// 16-element aligned: 16-byte loads / stores, 4 vectors in flight per thread.
__global__ void __launch_bounds__(kThreads) k_replica_gather(const Tile* __restrict__ tiles, int ntiles, PeerPtrs res,
                                                             float* __restrict__ grad, bool acc) {
  pdl_wait();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const float* src = reinterpret_cast<const float*>(res.p[tl.pad]) + tl.dst;
    float* g = grad + tl.dst;
    const uint32_t n = tl.n, nv = n / 4;
    constexpr uint32_t U = 4;
    uint32_t v = threadIdx.x;
    for (; v + (U - 1) * kThreads < nv; v += U * kThreads) {
      uint4 x[U];
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) x[u] = ld_stream(src + 4 * (v + u * kThreads));
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) {
        float4* gp = reinterpret_cast<float4*>(g) + v + u * kThreads;
        float4 y = make_float4(__uint_as_float(x[u].x), __uint_as_float(x[u].y), __uint_as_float(x[u].z),
                               __uint_as_float(x[u].w));
        if (acc) {
          const float4 o = *gp;
          y = make_float4(__fadd_rn(o.x, y.x), __fadd_rn(o.y, y.y), __fadd_rn(o.z, y.z), __fadd_rn(o.w, y.w));
        }
        *gp = y;
      }
    }
    for (; v < nv; v += kThreads) {
      const uint4 x = ld_stream(src + 4 * v);
      float4* gp = reinterpret_cast<float4*>(g) + v;
      float4 y = make_float4(__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z), __uint_as_float(x.w));
      if (acc) {
        const float4 o = *gp;
        y = make_float4(__fadd_rn(o.x, y.x), __fadd_rn(o.y, y.y), __fadd_rn(o.z, y.z), __fadd_rn(o.w, y.w));
      }
      *gp = y;
    }
    for (uint32_t e = nv * 4 + threadIdx.x; e < n; e += kThreads) g[e] = acc ? __fadd_rn(g[e], src[e]) : src[e];
  }
}

}  // namespace

cudaError_t launch_replica_gather(const Tile* tiles, int ntiles, PeerPtrs res, float* grad, bool accumulate,
                                  fsdpk::LaunchCfg cfg, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  if (cfg.variant & 2) {   // TMA bulk: the single-source pull with per-tile source (tile.src = tile.dst)
    const PullOps ops = make_ops(1, false, accumulate, false, cfg);
    return launch_pull_bulk_w<1, false, 1, true>(tiles, ntiles, res, grad, ops, grid_for(ntiles, cfg), st, cfg.pdl);
  }
  return launch_p(cfg.pdl, k_replica_gather, grid_for(ntiles, cfg), 0, st, tiles, ntiles, res, grad, accumulate);
}

cudaError_t launch_rs_pull_nested(const Tile* tiles, int ntiles, PeerPtrs staging, bool grad_bf16, int divisor,
                                  float* grad, bool mean, bool accumulate, bool bf16_reduce, int W, int G,
                                  fsdpk::LaunchCfg cfg, cudaStream_t st) {
  if (G == W)
    return launch_rs_pull(tiles, ntiles, staging, grad_bf16, divisor, grad, mean, accumulate, bf16_reduce, W, cfg, st);
  if (ntiles == 0) return cudaSuccess;
  const PullOps ops = make_ops(divisor, mean, accumulate, bf16_reduce, cfg);
  const int g = grid_for(ntiles, cfg);
  return grad_bf16 ? launch_nested<true>(tiles, ntiles, staging, grad, ops, W, G, g, st, cfg.variant, cfg.pdl)
                   : launch_nested<false>(tiles, ntiles, staging, grad, ops, W, G, g, st, cfg.variant, cfg.pdl);
}

}  // namespace fsdpp
