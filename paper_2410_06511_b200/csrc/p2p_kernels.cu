// Fused peer-memory kernels (see p2p.h): unshard push, reduce-scatter pull, the
// signal/wait handshake and the grad staging gather.  sm_100a, no fast math.
#include "p2p.h"

#include "dev_util.cuh"
#include "p2p_pull.cuh"

namespace fsdpp {
namespace {

using namespace fsdpdev;
using fsdpk::Tile;

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------- handshake
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The spin is bounded: after timeout_ns without the peer's flag (a rank that skipped the
// collective, or died) the kernel records {kind=2 (timeout), peer} in *err and returns, so a
// protocol error surfaces as FSDP_ERR_TIMEOUT from fsdp_mesh_synchronize instead of a hang.
__global__ void k_signal_wait(FlagPtrs remote, unsigned long long* local, int W, int rank,
                              unsigned long long* epoch_ctr, unsigned long long timeout_ns, int* err, int fence) {
  __shared__ unsigned long long e_sh;
  pdl_wait();   // launched programmatically after the data kernel (done handshakes)
  const int r = threadIdx.x;
  if (r == 0) {
    e_sh = *epoch_ctr + 1;
    *epoch_ctr = e_sh;
  }
  // A system-scope fence, on one thread, before the signal exactly where the protocol
  // publishes data that unfenced local kernels wrote and peers read next (`fence`, chosen
  // per call site: the pull's / world pull's ready (staging or zero-copy grads written by
  // the caller's or the staging kernel), the two-phase HSDP done (the result pieces), the
  // P2P amax all-reduce's ready (the amax copy), copy-engine transfers).  It orders that data
  // (cumulatively, through the CTA barrier and the signalling thread's release store) before
  // the flag.  Elsewhere the data a peer reads next was stored by a kernel that ends with its
  // own system fence (push, store-scatter) or there is none (a buffer handed back after
  // reads, which completed with the kernel that made them).  After the wait nothing needs a
  // fence: peers released their data before their flags, ld.acquire.sys observes the flags,
  // and the consumers are later kernels on this GPU.  Measured (profiles/round2/r2fence):
  // one fence per handshake on both sides cost 35% of a small unit's step (toy W=2 CUDA
  // graph 90 -> 122 us) and 1.2% of the 8B step.  -DFSDP_HS_FENCE fences every handshake on
  // both sides (debugging).
#ifdef FSDP_HS_FENCE
  fence = 1;
#endif
  if (fence && r == 0) __threadfence_system();
  __syncthreads();
  const unsigned long long epoch = e_sh;
#pragma unroll
  for (int i = 0; i < kMaxRanks; ++i)   // constant indices: remote.p stays in param space
    if (i == r && i < W) st_release_sys(remote.p[i] + rank, epoch);
  if (r < W) {
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(local + r) < epoch) {
      __nanosleep(64);
      if (globaltimer_ns() - t0 > timeout_ns) {
        { *(volatile int*)err = 2 | (r << 8); __threadfence_system(); }
        break;
      }
    }
  }
  __syncthreads();
#ifdef FSDP_HS_FENCE
  if (r == 0) __threadfence_system();
#endif
}

// Delayed-scaling amax fused into the fp8 cast: every thread keeps the
// max |x| bit pattern of the fp32 elements it cast (non-negative fp32 bits order like
// uint32; NaN patterns propagate), the warp reduces it and lane 0 folds it into
// acc[param] with atomicMax — the same uint-bit max as K1, so the result is bit-identical.
__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }
// One atomic per CTA per tile: warp max -> shared -> warp 0 max -> thread 0 atomicMax
// (~13K atomics per 8B block instead of ~106K per-warp ones, which serialised at L2 on the
// ~7 addresses of a block and cost ~80 us).  A running per-param max committed only when the
// param changes needed 24 more registers (64) and cut the push's occupancy.  CTA-uniform
// call; red[] is reused after the trailing barrier.
__device__ __forceinline__ void amax_commit_cta(uint32_t* acc, uint32_t param, uint32_t m, uint32_t* red) {
  m = __reduce_max_sync(0xFFFFFFFFu, m);
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t r = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0u;
    r = __reduce_max_sync(0xFFFFFFFFu, r);
    if (threadIdx.x == 0 && r) atomicMax(acc + param, r);
  }
  __syncthreads();
}
// ------------------------------------------------------------------- unshard push
template <int V>   // floats per 16-byte output vector: 8 (bf16) or 16 (e4m3)
__device__ __forceinline__ void load_floats(const float* p, uint32_t ph, float (&x)[V]) {
  // p = aligned base (16 B); the V floats start at word ph (0..3)
  constexpr int NQ = V / 4 + 1;
  float w[NQ * 4];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    if (i < V / 4 || ph != 0) {
      const uint4 q = ld_stream(p + 4 * i);
      w[4 * i] = __uint_as_float(q.x); w[4 * i + 1] = __uint_as_float(q.y);
      w[4 * i + 2] = __uint_as_float(q.z); w[4 * i + 3] = __uint_as_float(q.w);
    }
  }
  switch (ph) {
    case 0:
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = w[i];
      break;
    case 1:
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = w[i + 1];
      break;
    case 2:
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = w[i + 2];
      break;
    default:
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = w[i + 3];
      break;
  }
}

// load_floats + max |x| bits of the V selected words, taken on the loaded words before the
// phase shift (a per-word mask instead of a max after it: that variant needed 18 more registers)
template <int V>
__device__ __forceinline__ void load_floats_amax(const float* p, uint32_t ph, float (&x)[V], uint32_t& am) {
  constexpr int NQ = V / 4 + 1;
  float w[NQ * 4];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    if (i < V / 4 || ph != 0) {
      const uint4 q = ld_stream(p + 4 * i);
      w[4 * i] = __uint_as_float(q.x); w[4 * i + 1] = __uint_as_float(q.y);
      w[4 * i + 2] = __uint_as_float(q.z); w[4 * i + 3] = __uint_as_float(q.w);
    } else {
      w[4 * i] = w[4 * i + 1] = w[4 * i + 2] = w[4 * i + 3] = 0.0f;
    }
  }
#pragma unroll
  for (int i = 0; i < NQ * 4; ++i)
    if ((uint32_t)i >= ph && (uint32_t)i < ph + V) am = max(am, __float_as_uint(w[i]) & 0x7FFFFFFFu);
  switch (ph) {
    case 0:
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = w[i];
      break;
    case 1:
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = w[i + 1];
      break;
    case 2:
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = w[i + 2];
      break;
    default:
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = w[i + 3];
      break;
  }
}

__device__ __forceinline__ uint4 cvt_bf16x8(const float (&x)[8]) {
  return make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]),
                    pack_bf16x2(x[6], x[7]));
}
__device__ __forceinline__ uint4 cvt_e4m3x16(const float (&x)[16], float s) {
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t lo = pack_e4m3x2(__fmul_rn(x[4 * j], s), __fmul_rn(x[4 * j + 1], s));
    const uint32_t hi = pack_e4m3x2(__fmul_rn(x[4 * j + 2], s), __fmul_rn(x[4 * j + 3], s));
    w[j] = lo | (hi << 16);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <bool kFp8, bool kAmax = false>
__device__ __forceinline__ void push_tile(const Tile& tl, const float* __restrict__ shard, float s,
                                          const PeerPtrs& arena, int W, int rank, uint32_t* amp = nullptr) {
  uint32_t am = 0;
  constexpr uint32_t es = kFp8 ? 1 : 2;
  constexpr uint32_t V = 16 / es;
  const float* src = shard + tl.src;
  const uint64_t dst0 = tl.dst;
  const uint32_t n = tl.n;
  uint32_t h = (uint32_t)(((16u - (uint32_t)(dst0 & 15u)) & 15u) / es);
  if (h > n) h = n;
  const uint32_t nb = (n - h) / V;
  const uint32_t ph = h & 3u;
  const float* abase = src + (h - ph);
  // body: full 16-byte vectors, stored to every rank's arena; two vectors per thread per
  // iteration so both vectors' loads are in flight before the stores
  uint32_t v = threadIdx.x;
  for (; v + kThreads < nb; v += 2 * kThreads) {
    float x0[V], x1[V];
    if constexpr (kAmax) {
      load_floats_amax<V>(abase + V * v, ph, x0, am);
      load_floats_amax<V>(abase + V * (v + kThreads), ph, x1, am);
    } else {
      load_floats<V>(abase + V * v, ph, x0);
      load_floats<V>(abase + V * (v + kThreads), ph, x1);
    }
    uint4 o0, o1;
    if constexpr (kFp8) { o0 = cvt_e4m3x16(x0, s); o1 = cvt_e4m3x16(x1, s); }
    else { o0 = cvt_bf16x8(x0); o1 = cvt_bf16x8(x1); }
    const uint64_t off0 = dst0 + (uint64_t)h * es + 16ull * v;
    const uint64_t off1 = off0 + 16ull * kThreads;
    // arena.p is pre-rotated on the host (p[i] = rank (rank+1+i) % W's arena) so every rank
    // starts on a different peer; constant indices keep the pointers out of local memory
#pragma unroll
    for (int i = 0; i < kMaxRanks; ++i) {
      if (i >= W) break;
      st_v4(arena.p[i] + off0, o0);
      st_v4(arena.p[i] + off1, o1);
    }
  }
  for (; v < nb; v += kThreads) {
    float x[V];
    if constexpr (kAmax) load_floats_amax<V>(abase + V * v, ph, x, am);
    else load_floats<V>(abase + V * v, ph, x);
    uint4 o;
    if constexpr (kFp8) o = cvt_e4m3x16(x, s);
    else o = cvt_bf16x8(x);
    const uint64_t off = dst0 + (uint64_t)h * es + 16ull * v;
#pragma unroll
    for (int i = 0; i < kMaxRanks; ++i) {
      if (i >= W) break;
      st_v4(arena.p[i] + off, o);
    }
  }
  // head and tail elements (partial 16-byte vectors: element-sized stores only)
  const uint32_t tail0 = h + nb * V;
  for (uint32_t e = threadIdx.x; e < h + (n - tail0); e += kThreads) {
    const uint32_t el = e < h ? e : tail0 + (e - h);
    const uint64_t off = dst0 + (uint64_t)el * es;
    if (kFp8) {
      if constexpr (kAmax) am = max(am, abs_bits(src[el]));
      const uint8_t b = (uint8_t)(pack_e4m3x2(__fmul_rn(src[el], s), 0.0f) & 0xFFu);
#pragma unroll
      for (int d = 0; d < kMaxRanks; ++d) {
        if (d >= W) break;
        arena.p[d][off] = b;
      }
    } else {
      const uint16_t b = (uint16_t)(pack_bf16x2(src[el], 0.0f) & 0xFFFFu);
#pragma unroll
      for (int d = 0; d < kMaxRanks; ++d) {
        if (d >= W) break;
        *reinterpret_cast<uint16_t*>(arena.p[d] + off) = b;
      }
    }
  }
  if constexpr (kAmax) *amp = max(*amp, am);
}

// kAmax is a template parameter, not a runtime branch: with both fp8 paths in one kernel the
// register count doubled (37 -> 79 bulk, 56 -> 106 register push), occupancy fell and the bf16
// W=1 step went 15.2 -> 18.3 ms (profiles/round2/v2).  The amax-free instance is the old kernel.
template <bool kAmax>
__global__ void __launch_bounds__(kThreads) k_unshard_push(const Tile* __restrict__ tiles, int ntiles,
                                                           const float* __restrict__ shard,
                                                           const float* __restrict__ scales, PeerPtrs arena,
                                                           int W, int rank, uint32_t* __restrict__ acc) {
  __shared__ uint32_t red[kThreads / 32];
  pdl_wait();   // the ready handshake before it has completed
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    if (tl.kind == fsdpk::TK_FP8) {
      if constexpr (kAmax) {
        uint32_t mm = 0;
        push_tile<true, true>(tl, shard, scales[tl.param], arena, W, rank, &mm);
        amax_commit_cta(acc, tl.param, mm, red);
      } else {
        push_tile<true>(tl, shard, scales[tl.param], arena, W, rank);
      }
    }
    else push_tile<false>(tl, shard, 0.0f, arena, W, rank);
  }
  __threadfence_system();
}

// ------------------------------------------------------------------- store RS, own rows direct
// Receiver of the store-based reduce-scatter reading this rank's OWN rows straight from its
// full grads instead of from an own receive slot the scatter would have copied them into
// (saves 4 bytes of HBM per own bf16 element).  Source q is slot q of the local
// receive buffer for q != me and the caller's grads for q == me; the arithmetic is the pull's
// (every term / divisor, ascending-rank fp32 sum), so the bits are identical.  All sources are
// local HBM and 16-byte aligned (tile dst = off_p + j; own source checked by the caller):
// 16-byte loads, 8 elements per thread per vector (pull_body8).
template <int W, bool kGradBf16>
__global__ void __launch_bounds__(kThreads) k_rs_reduce_own(const Tile* __restrict__ tiles, int ntiles,
                                                            const uint8_t* recv, uint64_t slot_bytes,
                                                            fsdpk::PtrArray own, int me, float* __restrict__ grad,
                                                            PullOps ops) {
  constexpr uint32_t gs = kGradBf16 ? 2 : 4;
  pdl_wait();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const uint64_t sb = tl.dst * gs;   // byte offset in every receive slot
    const uintptr_t ownp = (uintptr_t)own.p[tl.param] + tl.src * gs;
    PeerPtrs st;
#pragma unroll
    for (int q = 0; q < W; ++q)   // st.p[q] + sb = the address of source q's rows
      st.p[q] = (q == me) ? (uint8_t*)(ownp - sb) : const_cast<uint8_t*>(recv) + (uint64_t)q * slot_bytes;
    float* g = grad + tl.dst;
    const uint32_t n = tl.n;
    const uint32_t nv = n / 8;
    pull_body8<W, kGradBf16, true>(st, sb, g, nv, 0, ops);
    for (uint32_t e = nv * 8 + threadIdx.x; e < n; e += kThreads) {
      float a = 0.0f;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const uint8_t* p = st.p[q] + sb + (uint64_t)gs * e;
        const float x = kGradBf16 ? __uint_as_float(((uint32_t)(*(const uint16_t*)p)) << 16) : *(const float*)p;
        const float y = ops.rb(ops.div(x));
        a = q == 0 ? y : __fadd_rn(a, y);
      }
      a = ops.rb(a);
      g[e] = ops.acc ? __fadd_rn(g[e], a) : a;
    }
  }
}

// ------------------------------------------------------------------- TMA bulk variants
// Pull: the TMA engine brings each rank's chunk (LaunchCfg::pull_chunk, 4 KB default) of the
// tile into shared memory (cp.async.bulk global->shared, mbarrier complete_tx, pull_stages
// stages), threads reduce from smem.
// Push: threads cast a 4 KB output chunk into smem once, one thread bulk-stores it into
// every rank's arena (cp.async.bulk shared->global, W stores per chunk, 2 stages).
constexpr uint32_t kBulkChunk = 4096;
static_assert(kBulkChunk / 16 == (uint32_t)kThreads, "push_tile_bulk: one 16-byte vector per thread per chunk");
template <bool kFp8, bool kAmax = false, bool kPref = false, int NSTG = 2>
__device__ __forceinline__ void push_tile_bulk(const Tile& tl, const float* __restrict__ shard, float s,
                                               const PeerPtrs& arena, int W, uint8_t* stage_buf, uint32_t& it,
                                               uint32_t* amp = nullptr) {
  uint32_t am = 0;
  constexpr uint32_t es = kFp8 ? 1 : 2;
  constexpr uint32_t V = 16 / es;                    // elements per 16-byte vector
  constexpr uint32_t CV = kBulkChunk / 16;           // vectors per chunk (= kThreads)
  const float* src = shard + tl.src;
  const uint64_t dst0 = tl.dst;
  const uint32_t n = tl.n;
  uint32_t h = (uint32_t)(((16u - (uint32_t)(dst0 & 15u)) & 15u) / es);
  if (h > n) h = n;
  const uint32_t nb = (n - h) / V;
  const uint32_t ph = h & 3u;
  const float* abase = src + (h - ph);
  const uint64_t body0 = dst0 + (uint64_t)h * es;   // 16-byte aligned
  const uint32_t nch = (nb + CV - 1) / CV;
  // kPref (the bf16-only kernel): register double buffer — chunk c+1's loads are in flight
  // across chunk c's barriers and bulk-store issue (the mixed fp8 kernels keep one buffer:
  // a second one would cost 8-16 registers and their 6-CTA/SM occupancy)
  auto load_chunk = [&](uint32_t c, float (&x)[V]) -> bool {
    const uint32_t v = c * CV + threadIdx.x;
    if (v >= nb) return false;
    if constexpr (kAmax) load_floats_amax<V>(abase + V * v, ph, x, am);
    else load_floats<V>(abase + V * v, ph, x);
    return true;
  };
  float xn[V];
  bool hn = kPref && nch > 0 && load_chunk(0, xn);
  for (uint32_t c = 0; c < nch; ++c, ++it) {
    uint8_t* buf = stage_buf + (size_t)(it % NSTG) * kBulkChunk;
    float x[V];
    bool hx;
    if constexpr (kPref) {
#pragma unroll
      for (uint32_t i = 0; i < V; ++i) x[i] = xn[i];
      hx = hn;
      if (c + 1 < nch) hn = load_chunk(c + 1, xn);
    }
    if (threadIdx.x == 0) bulk_wait_read_le<NSTG - 1>();   // the chunk written NSTG iterations ago was read
    __syncthreads();
    if constexpr (!kPref) hx = load_chunk(c, x);
    if (hx) {
      uint4 o;
      if constexpr (kFp8) o = cvt_e4m3x16(x, s);
      else o = cvt_bf16x8(x);
      *reinterpret_cast<uint4*>(buf + 16 * threadIdx.x) = o;
    }
    fence_proxy_async_smem();                         // generic smem writes -> async proxy
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = 16u * min(CV, nb - c * CV);
#pragma unroll
      for (int d = 0; d < kMaxRanks; ++d) {
        if (d >= W) break;
        bulk_s2g(arena.p[d] + body0 + (uint64_t)c * kBulkChunk, buf, bytes);
      }
      bulk_commit();
    }
  }
  // head and tail elements (partial 16-byte vectors: element-sized stores only)
  const uint32_t tail0 = h + nb * V;
  for (uint32_t e = threadIdx.x; e < h + (n - tail0); e += kThreads) {
    const uint32_t el = e < h ? e : tail0 + (e - h);
    const uint64_t off = dst0 + (uint64_t)el * es;
    if (kFp8) {
      if constexpr (kAmax) am = max(am, abs_bits(src[el]));
      const uint8_t b = (uint8_t)(pack_e4m3x2(__fmul_rn(src[el], s), 0.0f) & 0xFFu);
#pragma unroll
      for (int d = 0; d < kMaxRanks; ++d) {
        if (d >= W) break;
        arena.p[d][off] = b;
      }
    } else {
      const uint16_t b = (uint16_t)(pack_bf16x2(src[el], 0.0f) & 0xFFFFu);
#pragma unroll
      for (int d = 0; d < kMaxRanks; ++d) {
        if (d >= W) break;
        *reinterpret_cast<uint16_t*>(arena.p[d] + off) = b;
      }
    }
  }
  if constexpr (kAmax) *amp = max(*amp, am);
}

// kAnyFp8 = false: the bf16 unshard (every tile TK_BF16) — only the bf16 path is compiled, so
// the register double buffer fits in 31 registers and 8 CTAs per SM (kCtasPushW1: the push
// alone 245.7 -> 238.5 us per 8B block, profiles/round2/r2pref bench_cta8)
constexpr int kCtasPushW1 = 8;
#ifndef FSDP_PUSH_W1_STAGES
#define FSDP_PUSH_W1_STAGES 2
#endif
constexpr int kPushW1Stages = FSDP_PUSH_W1_STAGES;   // smem output stages of the bf16-only push
template <bool kAmax, bool kAnyFp8 = true>
__global__ void __launch_bounds__(kThreads) k_unshard_push_bulk(const Tile* __restrict__ tiles, int ntiles,
                                                                const float* __restrict__ shard,
                                                                const float* __restrict__ scales, PeerPtrs arena,
                                                                int W, uint32_t* __restrict__ acc) {
  // the bf16-only W = 1 instance keeps kPushW1Stages output chunks in flight (FSDP_B200 A/B:
  // profiles/round2); the mixed fp8 instances keep 2
  constexpr int NSTG = kAnyFp8 ? 2 : kPushW1Stages;
  __shared__ __align__(128) uint8_t stage_buf[NSTG * kBulkChunk];
  __shared__ uint32_t red[kThreads / 32];
  pdl_wait();
  uint32_t it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    if (kAnyFp8 && tl.kind == fsdpk::TK_FP8) {
      if constexpr (kAmax) {
        uint32_t mm = 0;
        push_tile_bulk<true, true>(tl, shard, scales[tl.param], arena, W, stage_buf, it, &mm);
        amax_commit_cta(acc, tl.param, mm, red);
      } else if constexpr (kAnyFp8) {
        push_tile_bulk<true>(tl, shard, scales[tl.param], arena, W, stage_buf, it);
      }
    }
    else push_tile_bulk<false, false, !kAnyFp8, NSTG>(tl, shard, 0.0f, arena, W, stage_buf, it);
  }
  if (threadIdx.x == 0) bulk_wait0();                 // every bulk store has completed
  __syncthreads();
  __threadfence_system();
}

// ------------------------------------------------------------------- fp8 amax all-reduce(max)
// out[i] = max over the W ranks' copies of the amax bit patterns (uint32 max == fp32 max of
// non-negative values, NaN patterns propagate; the same reduction as ncclMax on uint32).
__global__ void __launch_bounds__(kThreads) k_amax_max(PeerPtrs src, int W, uint32_t* __restrict__ out, int n) {
  for (int i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) {
    uint32_t v = 0;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) {
      if (q >= W) break;
      v = max(v, reinterpret_cast<const uint32_t*>(src.p[q])[i]);
    }
    out[i] = v;
  }
}

// ------------------------------------------------------------------- W = 1 cast, TMA in / out
// The W = 1 unshard modelled on the 3-stage K5: per 2048-element chunk the TMA engine loads
// the fp32 rows into shared memory (mbarrier complete_tx, NS stages ahead), threads cast them
// into an output stage — 8 floats -> one 16-byte bf16 vector (TK_BF16 tiles), or 16 floats ->
// one 16-byte e4m3 vector with the param's scale (TK_FP8) — and one thread bulk-stores it.
// kAmax (delayed scaling, amax fused): max |x| bits of the TK_FP8 tiles, one atomic per CTA
// per tile, as the push.  Tiles whose fp32 source, destination or length are not 16-byte
// granular take an element path (none in the Llama layouts).  Tile: src = shard element
// offset, dst = byte offset into the arena, n elements (layout.h tiles_push).
constexpr uint32_t kCastChunk = 2048;
// W > 1 (FSDP_B200_VARIANT bit 128): the same kernel stores every output chunk into all W
// arenas (arena.p rotated per rank on the host), i.e. the push with TMA loads.
template <int NS, bool kAnyFp8, bool kAmax, bool kMulti = false>   // kMulti: W > 1 (bit 128)
__global__ void __launch_bounds__(kThreads) k_cast_w1_tma(const Tile* __restrict__ tiles, int ntiles,
                                                           const float* __restrict__ shard,
                                                           const float* __restrict__ scales,
                                                           PeerPtrs arena, int W, uint32_t* __restrict__ acc) {
  extern __shared__ __align__(128) uint8_t cast_smem[];   // [NS][chunk * 4] in, [NS][chunk * 2] out
  float (*sin)[kCastChunk] = reinterpret_cast<float (*)[kCastChunk]>(cast_smem);
  uint8_t (*sout)[kCastChunk * 2] = reinterpret_cast<uint8_t (*)[kCastChunk * 2]>(cast_smem + NS * kCastChunk * 4);
  __shared__ uint64_t full[NS];
  __shared__ uint32_t red[kThreads / 32];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  uint32_t it = 0;   // TMA chunks of this CTA: stage it % NS, parity (it / NS) & 1
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const float* s = shard + tl.src;
    const uint32_t n = tl.n;
    const bool f8 = kAnyFp8 && tl.kind == fsdpk::TK_FP8;   // CTA-uniform
    const float sc = f8 ? scales[tl.param] : 0.0f;
    uint32_t am = 0;
    if ((tl.src & 3u) != 0 || (tl.dst & 15u) != 0 || (n & 15u) != 0) {   // element path
      for (uint32_t e = threadIdx.x; e < n; e += kThreads) {
        if (f8) {
          if constexpr (kAmax) am = max(am, abs_bits(s[e]));
          const uint8_t b = (uint8_t)(pack_e4m3x2(__fmul_rn(s[e], sc), 0.0f) & 0xFFu);
          for (int q = 0; q < (kMulti ? W : 1); ++q) arena.p[q][tl.dst + e] = b;
        } else {
          const uint16_t b = (uint16_t)(pack_bf16x2(s[e], 0.0f) & 0xFFFFu);
          for (int q = 0; q < (kMulti ? W : 1); ++q) reinterpret_cast<uint16_t*>(arena.p[q] + tl.dst)[e] = b;
        }
      }
    } else {
      const uint32_t es = f8 ? 1u : 2u;   // output bytes per element
      const uint32_t nch = (n + kCastChunk - 1) / kCastChunk;
      auto issue = [&](uint32_t c) {   // thread 0: chunk c of this tile into stage (it + c) % NS
        const uint32_t i = it + c, st = i % NS;
        const uint32_t ne = min(kCastChunk, n - c * kCastChunk);
        mbar_arrive_expect_tx(&full[st], ne * 4);
        bulk_g2s(sin[st], s + (size_t)c * kCastChunk, ne * 4, &full[st]);
      };
      if (threadIdx.x == 0)
        for (uint32_t c = 0; c < (uint32_t)NS && c < nch; ++c) issue(c);
      for (uint32_t c = 0; c < nch; ++c) {
        const uint32_t i = it + c, st = i % NS;
        const uint32_t ne = min(kCastChunk, n - c * kCastChunk);
        mbar_wait(&full[st], (i / NS) & 1u);
        if (threadIdx.x == 0) bulk_wait_read_le<NS - 1>();   // sout[st] (stored NS chunks ago) was read
        __syncthreads();
        if (f8) {
          if constexpr (kAnyFp8) {
            for (uint32_t e16 = threadIdx.x; e16 * 16 < ne; e16 += kThreads) {
              float x[16];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 a = *reinterpret_cast<const float4*>(&sin[st][e16 * 16 + 4 * j]);
                x[4 * j] = a.x; x[4 * j + 1] = a.y; x[4 * j + 2] = a.z; x[4 * j + 3] = a.w;
              }
              if constexpr (kAmax) {
#pragma unroll
                for (int j = 0; j < 16; ++j) am = max(am, abs_bits(x[j]));
              }
              *reinterpret_cast<uint4*>(sout[st] + e16 * 16) = cvt_e4m3x16(x, sc);
            }
          }
        } else {
          for (uint32_t e8 = threadIdx.x; e8 * 8 < ne; e8 += kThreads) {
            const float4 a = *reinterpret_cast<const float4*>(&sin[st][e8 * 8]);
            const float4 b = *reinterpret_cast<const float4*>(&sin[st][e8 * 8 + 4]);
            *reinterpret_cast<uint4*>(sout[st] + e8 * 16) =
                make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
          }
        }
        fence_proxy_async_smem();
        __syncthreads();   // sout[st] complete, sin[st] consumed
        if (threadIdx.x == 0) {
#pragma unroll
          for (int q = 0; q < (kMulti ? kMaxRanks : 1); ++q) {   // constant indices: arena.p in param space
            if (q >= W) break;
            bulk_s2g(arena.p[q] + tl.dst + (size_t)c * kCastChunk * es, sout[st], ne * es);
          }
          bulk_commit();
          if (c + NS < nch) issue(c + NS);
        }
      }
      it += nch;
    }
    if constexpr (kAmax) {
      if (f8) amax_commit_cta(acc, tl.param, am, red);
    }
  }
  if (kMulti) {   // the peers' data before the done handshake's signal (W = 1: kernel end suffices)
    if (threadIdx.x == 0) bulk_wait0();
    __syncthreads();
    __threadfence_system();
  } else if (threadIdx.x == 0) {
    bulk_wait0();
  }
}

// ------------------------------------------------------------------- gather copy
__global__ void __launch_bounds__(kThreads) k_gather_copy(const Tile* __restrict__ tiles, int ntiles,
                                                          fsdpk::PtrArray srcs, uint8_t* __restrict__ dst_base) {
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const uint8_t* s = (const uint8_t*)srcs.p[tl.param] + tl.src;
    uint8_t* d = dst_base + tl.dst;
    uint32_t n = tl.n;
    uint32_t head = (uint32_t)((16u - ((uintptr_t)d & 15u)) & 15u);
    if (head > n) head = n;
    if (threadIdx.x < head) d[threadIdx.x] = s[threadIdx.x];
    s += head; d += head; n -= head;
    const uint32_t nv = n >> 4;
    const uint32_t k = (uint32_t)((uintptr_t)s & 15u);
    if (k == 0) copy_body<true>(s, d, nv, 0);
    else copy_body<false>(s, d, nv, k);
    for (uint32_t e = nv * 16 + threadIdx.x; e < n; e += kThreads) d[e] = s[e];
  }
}

// ------------------------------------------------------------------- store-based RS, sender
// Each tile copies this rank's full-grad rows of one destination rank's chunk (local reads,
// misaligned phases realigned like K4) into that rank's receive buffer over NVLink (16-byte
// stores: the store mechanism runs at ~700 GB/s both ways vs ~660 for loads,
// profiles/nvlink_ceiling.json).
__global__ void __launch_bounds__(kThreads) k_rs_scatter(const Tile* __restrict__ tiles, int ntiles,
                                                         fsdpk::PtrArray grads, PeerPtrs dests) {
  pdl_wait();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    uint8_t* base = nullptr;
#pragma unroll
    for (int i = 0; i < kMaxRanks; ++i)   // constant indices: dests stays in param space
      if (i == (int)tl.pad) base = dests.p[i];
    const uint8_t* s = (const uint8_t*)grads.p[tl.param] + tl.src;
    uint8_t* d = base + tl.dst;
    uint32_t n = tl.n;
    uint32_t head = (uint32_t)((16u - ((uintptr_t)d & 15u)) & 15u);
    if (head > n) head = n;
    if (threadIdx.x < head) d[threadIdx.x] = s[threadIdx.x];
    s += head; d += head; n -= head;
    const uint32_t nv = n >> 4;
    const uint32_t k = (uint32_t)((uintptr_t)s & 15u);
    if (k == 0) copy_body<true>(s, d, nv, 0);
    else copy_body<false>(s, d, nv, k);
    for (uint32_t e = nv * 16 + threadIdx.x; e < n; e += kThreads) d[e] = s[e];
  }
  __threadfence_system();
}


template <bool kGradBf16>
cudaError_t launch_reduce_own_w(const Tile* tiles, int ntiles, const uint8_t* recv, uint64_t slot_bytes,
                                const fsdpk::PtrArray& own, int me, float* grad, PullOps ops, int W, int g,
                                cudaStream_t s, bool pdl) {
  switch (W) {
#define FSDP_OWN_CASE(w) \
    case w: return launch_p(pdl, k_rs_reduce_own<w, kGradBf16>, g, 0, s, tiles, ntiles, recv, slot_bytes, own, me, grad, ops);
    FSDP_OWN_CASE(1) FSDP_OWN_CASE(2) FSDP_OWN_CASE(3) FSDP_OWN_CASE(4)
    FSDP_OWN_CASE(5) FSDP_OWN_CASE(6) FSDP_OWN_CASE(7) FSDP_OWN_CASE(8)
#undef FSDP_OWN_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_signal_wait(FlagPtrs remote, unsigned long long* local, int W, int rank,
                               unsigned long long* epoch_ctr, unsigned long long timeout_ns, int* err,
                               cudaStream_t st, bool pdl, bool fence) {
  const int f = fence ? 1 : 0;
  if (pdl) return launch_pdl(k_signal_wait, 1, 32, 0, st, remote, local, W, rank, epoch_ctr, timeout_ns, err, f);
  k_signal_wait<<<1, 32, 0, st>>>(remote, local, W, rank, epoch_ctr, timeout_ns, err, f);
  return cudaGetLastError();
}

static cudaError_t launch_cast_tma(const Tile* tiles, int ntiles, const float* shard, const float* scales,
                                   const PeerPtrs& a, int W, uint32_t* amax_acc, fsdpk::LaunchCfg cfg, cudaStream_t st);

cudaError_t launch_unshard_push(const Tile* tiles, int ntiles, const float* shard, const float* scales,
                                PeerPtrs arena, int W, int rank, fsdpk::LaunchCfg cfg, cudaStream_t st,
                                uint32_t* amax_acc) {
  if (ntiles == 0) return cudaSuccess;
  PeerPtrs rot{};   // destination order starts at the next rank: spreads NVLink traffic
  for (int i = 0; i < W; ++i) rot.p[i] = arena.p[(rank + 1 + i) % W];
  if (W > 1 && (cfg.variant & 128))   // the TMA-load push (FSDP_B200_VARIANT bit 128)
    return launch_cast_tma(tiles, ntiles, shard, scales, rot, W, amax_acc, cfg, st);
  const int g = grid_for(ntiles, cfg, fsdpk::kCtasPush);
  if (cfg.variant & 4)   // TMA bulk push
    // the bf16-only double-buffered kernel at W = 1 (HBM-bound: the W=1 8B step 15.21 ->
    // 15.00 ms, profiles/round2/r2pref); W > 1 is NVLink-bound and keeps the single buffer.
    // scales == NULL: a bf16 unshard (an fp8 unshard always has scales; the mixed kernel also
    // handles bf16-only tables, so a caller passing scales for bf16 stays correct)
    return amax_acc ? launch_p(cfg.pdl, k_unshard_push_bulk<true>, g, 0, st, tiles, ntiles, shard, scales, rot, W, amax_acc)
           : (scales || W > 1)
               ? launch_p(cfg.pdl, k_unshard_push_bulk<false>, g, 0, st, tiles, ntiles, shard, scales, rot, W, amax_acc)
                    : launch_p(cfg.pdl, k_unshard_push_bulk<false, false>, grid_for(ntiles, cfg, kCtasPushW1), 0, st,
                               tiles, ntiles, shard, scales, rot, W, amax_acc);
  return amax_acc ? launch_p(cfg.pdl, k_unshard_push<true>, g, 0, st, tiles, ntiles, shard, scales, rot, W, rank, amax_acc)
                  : launch_p(cfg.pdl, k_unshard_push<false>, g, 0, st, tiles, ntiles, shard, scales, rot, W, rank, amax_acc);
}

cudaError_t launch_rs_pull(const Tile* tiles, int ntiles, PeerPtrs staging, bool grad_bf16, int divisor, float* grad, bool mean,
                           bool accumulate, bool bf16_reduce, int W, fsdpk::LaunchCfg cfg, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  const PullOps ops = make_ops(divisor, mean, accumulate, bf16_reduce, cfg);
  const int g = grid_for(ntiles, cfg);
  return grad_bf16 ? launch_pull_w<true>(tiles, ntiles, staging, grad, ops, W, g, st, cfg.variant, cfg.pdl)
                   : launch_pull_w<false>(tiles, ntiles, staging, grad, ops, W, g, st, cfg.variant, cfg.pdl);
}

static cudaError_t launch_cast_tma(const Tile* tiles, int ntiles, const float* shard, const float* scales,
                                   const PeerPtrs& a, int W, uint32_t* amax_acc, fsdpk::LaunchCfg cfg, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  constexpr int NS = 3;
  constexpr size_t smem = (size_t)NS * kCastChunk * (4 + 2);   // 36 KB
  const int g = grid_for(ntiles, cfg, fsdpk::kCtasCopy);
  if (W > 1) {
    if (amax_acc)
      return launch_p(cfg.pdl, k_cast_w1_tma<NS, true, true, true>, g, smem, st, tiles, ntiles, shard, scales, a, W,
                      amax_acc);
    if (scales)
      return launch_p(cfg.pdl, k_cast_w1_tma<NS, true, false, true>, g, smem, st, tiles, ntiles, shard, scales, a, W,
                      amax_acc);
    return launch_p(cfg.pdl, k_cast_w1_tma<NS, false, false, true>, g, smem, st, tiles, ntiles, shard, scales, a, W,
                    amax_acc);
  }
  if (amax_acc)
    return launch_p(cfg.pdl, k_cast_w1_tma<NS, true, true>, g, smem, st, tiles, ntiles, shard, scales, a, W, amax_acc);
  if (scales)
    return launch_p(cfg.pdl, k_cast_w1_tma<NS, true, false>, g, smem, st, tiles, ntiles, shard, scales, a, W, amax_acc);
  return launch_p(cfg.pdl, k_cast_w1_tma<NS, false, false>, g, smem, st, tiles, ntiles, shard, scales, a, W, amax_acc);
}

cudaError_t launch_cast_w1(const Tile* tiles, int ntiles, const float* shard, const float* scales, void* arena,
                           uint32_t* amax_acc, fsdpk::LaunchCfg cfg, cudaStream_t st) {
  PeerPtrs a{};
  a.p[0] = (uint8_t*)arena;
  return launch_cast_tma(tiles, ntiles, shard, scales, a, 1, amax_acc, cfg, st);
}

cudaError_t launch_amax_max(PeerPtrs src, int W, uint32_t* out, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int g = std::min((n + kThreads - 1) / kThreads, 148);
  k_amax_max<<<g, kThreads, 0, st>>>(src, W, out, n);
  return cudaGetLastError();
}

cudaError_t launch_gather_copy(const Tile* tiles, int ntiles, const fsdpk::PtrArray& srcs, void* dst,
                               fsdpk::LaunchCfg cfg, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  return launch_persistent(k_gather_copy, grid_for(ntiles, cfg), 0, st, tiles, ntiles, srcs, (uint8_t*)dst);
}

cudaError_t launch_rs_scatter(const Tile* tiles, int ntiles, const fsdpk::PtrArray& grads, PeerPtrs dests,
                              fsdpk::LaunchCfg cfg, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  return launch_p(cfg.pdl, k_rs_scatter, grid_for(ntiles, cfg, fsdpk::kCtasPush), 0, st, tiles, ntiles, grads,
                           dests);
}

cudaError_t launch_rs_reduce_own(const Tile* tiles, int ntiles, const void* recv, int64_t S, bool grad_bf16,
                                const fsdpk::PtrArray& own, int me, int divisor, float* grad, bool mean, bool accumulate,
                                bool bf16_reduce, int W, fsdpk::LaunchCfg cfg, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  const PullOps ops = make_ops(divisor, mean, accumulate, bf16_reduce, cfg);
  const int g = grid_for(ntiles, cfg);
  const uint64_t slot_bytes = (uint64_t)S * (grad_bf16 ? 2 : 4);
  return grad_bf16 ? launch_reduce_own_w<true>(tiles, ntiles, (const uint8_t*)recv, slot_bytes, own, me, grad, ops, W, g,
                                               st, cfg.pdl)
                   : launch_reduce_own_w<false>(tiles, ntiles, (const uint8_t*)recv, slot_bytes, own, me, grad, ops, W,
                                                g, st, cfg.pdl);
}

}  // namespace fsdpp
