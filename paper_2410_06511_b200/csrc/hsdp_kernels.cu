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

}  // namespace

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
