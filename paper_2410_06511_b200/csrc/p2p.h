// Fused peer-memory (NVLink / NVSwitch) kernels of the unshard and the gradient
// reduce-scatter (the paper's SymmetricMemory idea, P:147 / P:537,
// applied to FSDP's collectives).  Buffers are symmetric: every rank allocates the same
// sizes and maps its peers' copies with CUDA IPC, so a kernel can load/store any rank's
// buffer directly.
//
//   unshard:  k_signal_wait(ready) -> k_unshard_push -> k_signal_wait(done)
//             each rank casts its fp32 shard once (bf16 / e4m3 with per-tensor scale) and
//             stores the result into EVERY rank's unsharded-parameter arena at its rows:
//             copy-in + all-gather + copy-out in one kernel, no staging buffer.
//   reduce:   k_gather_copy (caller grads -> own symmetric staging, skipped if the caller
//             wrote there) -> k_signal_wait(ready) -> k_rs_pull -> k_signal_wait(done)
//             each rank reads its row chunk from every rank's staged bf16 grads, divides
//             each by W and sums in ascending rank order in fp32: the fp32
//             reduce-scatter with bf16 (not fp32) bytes on the wire and a deterministic
//             order.
// Only the single-CTA signal/wait kernels spin; the data kernels never block SMs.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace fsdpp {

constexpr int kMaxRanks = 16;

struct PeerPtrs { uint8_t* p[kMaxRanks]; };
struct FlagPtrs { unsigned long long* p[kMaxRanks]; };

// epoch = ++*epoch_ctr (device counter of this flag slot: every rank runs the same sequence
// of handshakes per slot, so the epochs agree, and a replayed CUDA graph advances them).
// Thread r < W: st.release.sys flags_remote.p[r][my_rank] = epoch (signal rank r), after a
// system-scope fence; then every thread r < W spins (ld.acquire.sys) until
// flags_local[r] >= epoch (rank r signalled me).  One CTA.
// The spin gives up after timeout_ns and writes 2 | (peer << 8) to *err (FSDP_ERR_TIMEOUT).
// pdl: launch with programmatic stream serialization (the done handshakes, right after their
// data kernel on the same stream: the launch latency overlaps the data kernel's tail).
// fence: a system-scope fence before the signal, for call sites whose peers next read data
// that local kernels without their own system fence wrote (see k_signal_wait).
cudaError_t launch_signal_wait(FlagPtrs remote, unsigned long long* local, int W, int rank,
                               unsigned long long* epoch_ctr, unsigned long long timeout_ns, int* err,
                               cudaStream_t st, bool pdl = false, bool fence = false);

// Push tiles: src = element offset into the fp32 shard, dst = byte offset into the arena,
// n elements, kind TK_BF16 / TK_FP8 (scale = scales[param]).  Stores go to arena.p[d] for
// every rank d (d = rank is the local arena), rotated by rank to spread NVLink traffic.
// amax_acc != NULL (delayed scaling with the amax fused into the push): amax_acc[param] =
// max(amax_acc[param], max |x| bits) over the TK_FP8 tiles' elements (uint-bit max, as K1).
cudaError_t launch_unshard_push(const fsdpk::Tile* tiles, int ntiles, const float* shard,
                                const float* scales, PeerPtrs arena, int W, int rank,
                                fsdpk::LaunchCfg cfg, cudaStream_t st, uint32_t* amax_acc = nullptr);

// Pull tiles: src = element offset into every rank's staging, dst = element offset into the
// fp32 grad, n elements.  grad[dst+e] (+)= round?( sum_{q=0..W-1} (fp32(stage_q[src+e]) / W) ).
cudaError_t launch_rs_pull(const fsdpk::Tile* tiles, int ntiles, PeerPtrs staging, bool grad_bf16, int divisor,
                           float* grad, bool mean, bool accumulate, bool bf16_reduce, int W,
                           fsdpk::LaunchCfg cfg, cudaStream_t st);

// HSDP on one NVSwitch domain (hsdp_kernels.cu): the same pull over the W = R * G ranks of
// the world, staging.p[g] = global rank g's staging (g = replica * G + shard rank), summed in
// groups of G consecutive sources: grad[dst+e] (+)= round?( sum_{r<R} ( sum_{q<G}
// fp32(stage_{r*G+q}[src+e]) / divisor ) ), both sums ascending fp32 (the
// shard-group reduce-scatter, then the replica all-reduce; oracle HsdpWorld 'order').
// G == W is launch_rs_pull.  Pairs with W <= 8 and G | W.
cudaError_t launch_rs_pull_nested(const fsdpk::Tile* tiles, int ntiles, PeerPtrs staging, bool grad_bf16, int divisor,
                                  float* grad, bool mean, bool accumulate, bool bf16_reduce, int W, int G,
                                  fsdpk::LaunchCfg cfg, cudaStream_t st);

// HSDP two-phase reduce-scatter (hsdp_kernels.cu): phase 1 is launch_rs_pull_nested over the
// tiles of this replica's piece (layout.h split_pieces) writing into this rank's fp32 result
// buffer; phase 2 copies every piece q from replica q's result buffer res.p[q] (tile.pad = q)
// into the grad: grad[dst+e] (+)= res.p[pad][dst+e].  Tile dst 16-element aligned.
cudaError_t launch_replica_gather(const fsdpk::Tile* tiles, int ntiles, PeerPtrs res, float* grad, bool accumulate,
                                  fsdpk::LaunchCfg cfg, cudaStream_t st);

// W = 1 unshard with TMA loads and stores (3 stages of 2048 elements): the push tiles' rows
// of the fp32 shard cast into the local arena (tiles_push: TK_BF16 -> bf16, TK_FP8 -> e4m3
// with scales[param]; scales NULL = a bf16-only table).  amax_acc != NULL: the fused amax of
// the TK_FP8 tiles (as launch_unshard_push).
cudaError_t launch_cast_w1(const fsdpk::Tile* tiles, int ntiles, const float* shard, const float* scales,
                           void* arena, uint32_t* amax_acc, fsdpk::LaunchCfg cfg, cudaStream_t st);

// fp8 amax all-reduce over symmetric memory: out[i] = max_{q < W} src.p[q][i] (uint32 bit
// patterns of non-negative fp32 amaxes), i < n.
cudaError_t launch_amax_max(PeerPtrs src, int W, uint32_t* out, int n, cudaStream_t st);

// Gather copy: dst + tile.dst <- srcs.p[param] + tile.src, n bytes (any alignment).
cudaError_t launch_gather_copy(const fsdpk::Tile* tiles, int ntiles, const fsdpk::PtrArray& srcs,
                               void* dst, fsdpk::LaunchCfg cfg, cudaStream_t st);

// Store-based reduce-scatter, sender (layout.h tiles_scatter): dests.p[tile.pad] + tile.dst <-
// grads.p[param] + tile.src, n bytes; ends with a system-scope fence.  The receiver then
// reduces its [W][S] receive buffer with launch_rs_pull (every "peer" pointer local).
cudaError_t launch_rs_scatter(const fsdpk::Tile* tiles, int ntiles, const fsdpk::PtrArray& grads, PeerPtrs dests,
                              fsdpk::LaunchCfg cfg, cudaStream_t st);

// Store-based reduce-scatter, receiver reading its own rows from its full grads (layout.h
// tiles_recv_reduce_own): for q != me the rows come from slot q of recv ([W][S] grad
// elements), for q == me from own.p[param] + src; grad[dst+e] (+)= round?(sum_q fp32(x_q)/W).
// recv and every own source must be 16-byte aligned (the caller checks).
cudaError_t launch_rs_reduce_own(const fsdpk::Tile* tiles, int ntiles, const void* recv, int64_t S, bool grad_bf16,
                                const fsdpk::PtrArray& own, int me, int divisor, float* grad, bool mean,
                                bool accumulate, bool bf16_reduce, int W, fsdpk::LaunchCfg cfg, cudaStream_t st);

}  // namespace fsdpp
