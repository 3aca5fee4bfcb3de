// Internal kernel launchers of the FSDP2 Shard(0) hot path (not part of the C ABI).
// Every kernel is HBM-bound (no dense contraction, <= 0.2 flop/byte): 128-bit
// coalesced vector loads/stores, persistent grid = SMs x resident CTAs, tile tables
// built once per layer on the host for the ragged per-parameter segments.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fsdpk {

// One unit of work of a segmented kernel.  Offsets are relative to the bases passed to
// the launch (or to ptrs[param] when the kernel takes a pointer array).
struct Tile {
  uint64_t src;    // byte offset (copy-out, amax: absolute address) / element offset
  uint64_t dst;    // byte offset / element offset
  uint32_t n;      // bytes (copy-out) or elements
  uint32_t param;  // param index (pointer array / scale index)
  uint32_t kind;   // TileKind
  uint32_t pad;    // K5: number of valid source elements (<= n); the rest is zero-filled
};
static_assert(sizeof(Tile) == 32, "Tile must be 32 bytes");

enum TileKind : uint32_t { TK_COPY = 0, TK_FP8 = 2, TK_BF16 = 3 };

constexpr int kMaxPtrs = 512;  // pointers per launch (4 KB kernel parameter)
struct PtrArray { const void* p[kMaxPtrs]; };

constexpr uint32_t kTileElems = 16384;   // K3/K5/K1 tile size in elements
constexpr uint32_t kTileBytes = 65536;   // K4 tile size in bytes

struct LaunchCfg {
  int grid_cap;     // max CTAs when the kernel has no tuned value (SMs * 4)
  int sms = 148;    // multiprocessor count
  int per_sm = 0;   // > 0: FSDP_B200_CTAS_PER_SM override for every kernel
  // kernel-variant bit mask (FSDP_B200_VARIANT, default 78): 1 = 16-byte pull loads, 2 = TMA
  // bulk pull, 4 = TMA bulk push, 8 = TMA bulk RS copy-in (K5), 32 = W=1 bf16 unshard as one
  // contiguous K2 cast when the arena has the flat layout, 64 = W=1 bf16 unshard as the
  // TMA-in / TMA-out cast (k_cast_w1_tma), 128 = the same kernel as the W>1 push (slower)
  int variant = 0;
  // TMA bulk pull: bytes per peer per chunk (power of two, 1-16 KB) and pipeline stages (2-4)
  // (FSDP_B200_PULL_CHUNK / FSDP_B200_PULL_STAGES)
  int pull_chunk = 4096;
  int pull_stages = 2;
  // P2P data kernels and done handshakes launched with programmatic dependent launch
  // (FSDP_B200_PDL=0 disables)
  bool pdl = true;
  // TMA-bulk K5 pipeline stages (FSDP_B200_K5_STAGES: 2, 3 or 4; 3 measured best: the K5
  // kernel 242 -> 228 us per 8B block, the W=1 step 15.07 -> 14.66 ms, profiles/round2/r2k5)
  int k5_stages = 3;
  // persistent grid of a kernel whose measured best is `tuned` CTAs per SM
  int cap(int tuned) const { return sms * (per_sm > 0 ? per_sm : tuned); }
};

// CTAs per SM (256 threads each) measured best on B200 (profiles/r02, 8B layout)
constexpr int kCtasRsCopyIn = 2;
constexpr int kCtasPush = 6;
constexpr int kCtasCopy = 4;

// K2: slot[i] = bf16_rne(shard[i]) for i < S (S % 16 == 0, both 16B aligned).
cudaError_t launch_copy_in_bf16(const float* shard, void* slot, int64_t S, LaunchCfg cfg,
                                cudaStream_t st);
// K3: per tile: TK_FP8 -> e4m3fn(satfinite(rn(x * scales[param]))), TK_BF16 -> bf16.
// src = element offset into shard, dst = byte offset into slot.  amax_acc != NULL: also
// amax_acc[param] = max(amax_acc[param], max |x| bits) over the TK_FP8 tiles (delayed scaling).
cudaError_t launch_copy_in_fp8(const Tile* tiles, int ntiles, const float* shard, void* slot,
                               const float* scales, LaunchCfg cfg, cudaStream_t st,
                               uint32_t* amax_acc = nullptr);
// K1c delayed scaling with the amax fused into the fp8 casts: for every idx j: a = acc[j]
// (the max |x| the casts since the previous call saw; all ranks' by then, after the
// all-reduce(max)); record a into the history FIRST (hist[pos[j]] = a, pos advances; a
// history not yet initialised is filled with a), then scale[j] = fp32(448 / fp64(max(max(
// hist), 1e-12))); amax_out[j] = a; acc[j] = 0.  Recording the previous step's amax at the
// start of this call is the same history as K1b recording it at the end of the previous one.
cudaError_t launch_fp8_scale_delayed_fused(const int32_t* idx, int n, uint32_t* acc_bits, float* amax_out,
                                           float* scale_out, const uint8_t* eligible, float* hist, int32_t* pos,
                                           uint8_t* hist_init, int H, int hmax, int* err_flag, cudaStream_t st);
// K4: byte copy: ptrs.p[param] + dst <- ag + src, n bytes (any alignment).
cudaError_t launch_copy_out(const Tile* tiles, int ntiles, const void* ag, const PtrArray& outs,
                            LaunchCfg cfg, cudaStream_t st);
// K5: rs_in[dst + e] = e < pad ? cast(grads.p[param][src + e]) / W : 0, e < n.
// grad_bf16: grads are bf16 (else fp32); out_bf16: rs_in is bf16 (else fp32).
cudaError_t launch_rs_copy_in(const Tile* tiles, int ntiles, const PtrArray& grads, bool grad_bf16,
                              void* rs_in, bool out_bf16, bool mean, int world_size,
                              LaunchCfg cfg, cudaStream_t st);
// K6: grad[i] (+)= widen(rs_out[i]) for i < S.
cudaError_t launch_rs_copy_out(const void* rs_out, bool in_bf16, float* grad, bool accumulate,
                               int64_t S, LaunchCfg cfg, cudaStream_t st);
// K1: acc_bits[param] = max(acc_bits[param], max |x| bits) over tiles (src absolute).
cudaError_t launch_amax(const Tile* tiles, int ntiles, uint32_t* acc_bits, LaunchCfg cfg,
                        cudaStream_t st);
// K1b: for i in idx[0..n): a = acc[idx]; amax[idx] = a; scale[idx] = eligible ?
// fp32(448/fp64(max(a,1e-12))) : 0; non-finite -> scale 0, *err_flag = 1; acc[idx] = 0
// when reset_acc.
cudaError_t launch_fp8_scale(const int32_t* idx, int n, uint32_t* acc_bits, float* amax_out,
                             float* scale_out, const uint8_t* eligible, int* err_flag,
                             bool reset_acc, cudaStream_t st);
// K1b delayed scaling: for every idx j with eligible[j]: if the history
// hist[j*hmax .. +H) is not initialised, fill it with a = acc[j]; scale[j] = fp32(448 /
// fp64(max(max(hist), 1e-12))); then hist[pos[j]] = a, pos[j] = (pos[j]+1) % H ("updated
// after use").  amax_out[j] = a; acc[j] = 0.
cudaError_t launch_fp8_scale_delayed(const int32_t* idx, int n, uint32_t* acc_bits, float* amax_out,
                                     float* scale_out, const uint8_t* eligible, float* hist, int32_t* pos,
                                     uint8_t* hist_init, int H, int hmax, int* err_flag, cudaStream_t st);

}  // namespace fsdpk
