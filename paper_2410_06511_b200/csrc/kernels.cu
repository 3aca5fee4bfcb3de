// Hand-written sm_100a kernels of the FSDP2 per-parameter Shard(0) step.
//
//   K2 copy-in bf16   (P:417 bf16 all-gather; P:464 multi-tensor all-gather copy-in)
//   K3 copy-in fp8    (P:157 Float8 all-gather with per-tensor scales)
//   K4 copy-out       (rank-major all-gather output -> per-parameter tensors)
//   K5 RS copy-in     (P:466 single pre-division by W; P:544 fp32 reduce-scatter)
//   K6 RS copy-out    (accumulate / widen into the fp32 sharded gradient)
//   K1 amax, K1b scale (P:157 dynamic tensorwise scaling)
//
// All of it is HBM-bound streaming work, so no tensor cores: the design rules are
// 128-bit coalesced accesses, several independent 16-byte loads in flight per thread,
// persistent grids sized to the SM count, and per-layer tile tables so the ragged
// per-parameter segments become uniform ~64 KB work items.  Compiled without fast
// math: IEEE division, no flush-to-zero (bit-exactness vs the oracle depends on it).
#include "kernels.h"

#include <cuda_bf16.h>

#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "dev_util.cuh"

namespace fsdpk {
namespace {

using namespace fsdpdev;

// ------------------------------------------------------------------- K2 copy-in bf16
// 4 floats per thread per vector: each warp instruction loads 512 contiguous bytes and
// stores 256 contiguous bytes.
__global__ void __launch_bounds__(kThreads) k_copy_in_bf16(const float4* __restrict__ src,
                                                           uint2* __restrict__ dst, int64_t n4) {
  constexpr int U = 2 * kUnroll;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = ld_stream(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u)
      st_v2(dst + i + u * stride, make_uint2(pack_bf16x2(__uint_as_float(a[u].x), __uint_as_float(a[u].y)),
                                             pack_bf16x2(__uint_as_float(a[u].z), __uint_as_float(a[u].w))));
  }
  for (; i < n4; i += stride) {
    const uint4 a = ld_stream(src + i);
    st_v2(dst + i, make_uint2(pack_bf16x2(__uint_as_float(a.x), __uint_as_float(a.y)),
                              pack_bf16x2(__uint_as_float(a.z), __uint_as_float(a.w))));
  }
}

// ------------------------------------------------------------------- K3 copy-in fp8
template <bool kAmax>   // compile-time: the amax-free instance keeps its 32 registers
__global__ void __launch_bounds__(kThreads) k_copy_in_fp8(const Tile* __restrict__ tiles, int ntiles,
                                                          const float* __restrict__ shard,
                                                          uint8_t* __restrict__ slot,
                                                          const float* __restrict__ scales,
                                                          uint32_t* __restrict__ acc) {
  uint32_t run_m = 0;   // delayed scaling: running max |x| bits of run_p's tiles, committed on change
  int run_p = -1;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const float* src = shard + tl.src;   // 16-element aligned
    uint8_t* dst = slot + tl.dst;        // 16-byte aligned
    const uint32_t n = tl.n;
    if (tl.kind == TK_FP8) {
      const float s = scales[tl.param];
      const uint32_t nv = n / 16;
      if (kAmax && (int)tl.param != run_p) {   // CTA-uniform
        if (run_p >= 0) {
          const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, run_m);
          if ((threadIdx.x & 31u) == 0 && m) atomicMax(acc + run_p, m);
        }
        run_p = (int)tl.param;
        run_m = 0;
      }
      uint32_t am = 0;   // delayed scaling: max |x| bits of the cast elements (acc != NULL)
      for (uint32_t v = threadIdx.x; v < nv; v += kThreads) {
        uint4 q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) q[j] = ld_stream(src + 16 * v + 4 * j);
        if constexpr (kAmax) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            am = max(am, max(max(q[j].x & 0x7FFFFFFFu, q[j].y & 0x7FFFFFFFu),
                             max(q[j].z & 0x7FFFFFFFu, q[j].w & 0x7FFFFFFFu)));
        }
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t lo = pack_e4m3x2(__fmul_rn(__uint_as_float(q[j].x), s),
                                          __fmul_rn(__uint_as_float(q[j].y), s));
          const uint32_t hi = pack_e4m3x2(__fmul_rn(__uint_as_float(q[j].z), s),
                                          __fmul_rn(__uint_as_float(q[j].w), s));
          w[j] = lo | (hi << 16);
        }
        st_v4(dst + 16 * v, make_uint4(w[0], w[1], w[2], w[3]));
      }
      for (uint32_t e = nv * 16 + threadIdx.x; e < n; e += kThreads) {
        if constexpr (kAmax) am = max(am, __float_as_uint(src[e]) & 0x7FFFFFFFu);
        const float x = __fmul_rn(src[e], s);
        dst[e] = (uint8_t)(pack_e4m3x2(x, 0.0f) & 0xFFu);
      }
      run_m = max(run_m, am);
    } else {  // bf16 param inside a float8 unit
      const uint32_t nv = n / 8;
      uint16_t* d16 = reinterpret_cast<uint16_t*>(dst);
      for (uint32_t v = threadIdx.x; v < nv; v += kThreads) {
        const uint4 a = ld_stream(src + 8 * v), b = ld_stream(src + 8 * v + 4);
        uint4 o;
        o.x = pack_bf16x2(__uint_as_float(a.x), __uint_as_float(a.y));
        o.y = pack_bf16x2(__uint_as_float(a.z), __uint_as_float(a.w));
        o.z = pack_bf16x2(__uint_as_float(b.x), __uint_as_float(b.y));
        o.w = pack_bf16x2(__uint_as_float(b.z), __uint_as_float(b.w));
        st_v4(d16 + 8 * v, o);
      }
      for (uint32_t e = nv * 8 + threadIdx.x; e < n; e += kThreads)
        d16[e] = (uint16_t)(pack_bf16x2(src[e], 0.0f) & 0xFFFFu);
    }
  }
  if (kAmax && run_p >= 0) {
    const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, run_m);
    if ((threadIdx.x & 31u) == 0 && m) atomicMax(acc + run_p, m);
  }
}

// ------------------------------------------------------------------- K4 copy-out
__global__ void __launch_bounds__(kThreads) k_copy_out(const Tile* __restrict__ tiles, int ntiles,
                                                       const uint8_t* __restrict__ ag, PtrArray outs) {
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const uint8_t* s = ag + tl.src;
    uint8_t* d = (uint8_t*)outs.p[tl.param] + tl.dst;
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

// ------------------------------------------------------------------- K5 RS copy-in
struct DivW {
  float w, inv;
  bool pow2, mean;
  __device__ __forceinline__ float operator()(float x) const {
    if (!mean) return x;
    return pow2 ? __fmul_rn(x, inv) : __fdiv_rn(x, w);   // both equal IEEE x / W
  }
};

// 4 elements per thread per vector: a warp's load instruction covers 256 B (bf16) / 512 B
// (fp32) and its store instruction 512 B (fp32) / 256 B (bf16), both contiguous — no
// half-filled sectors (the 8-element mapping wrote 2 x 16 B per thread at a 32 B stride).
template <bool kOutBf16>
__device__ __forceinline__ void store4(uint8_t* d, const float (&y)[4]) {
  if (kOutBf16) st_v2(d, make_uint2(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3])));
  else st_v4(d, make_uint4(__float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]), __float_as_uint(y[3])));
}

template <bool kGradBf16, bool kOutBf16, bool kAligned>
__device__ __forceinline__ void rs_body(const uint8_t* s, uint8_t* d, uint32_t nv, uint32_t k, DivW div) {
  constexpr uint32_t gs = kGradBf16 ? 8 : 16;   // source bytes per 4 elements
  constexpr uint32_t os = kOutBf16 ? 8 : 16;    // output bytes per 4 elements
  constexpr int U = 2 * kUnroll;
  uint32_t v = threadIdx.x;
  for (; v + (U - 1) * kThreads < nv; v += U * kThreads) {
    float x[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) load4<kGradBf16, kAligned>(s + gs * (v + u * kThreads), k, x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int j = 0; j < 4; ++j) x[u][j] = div(x[u][j]);
      store4<kOutBf16>(d + os * (v + u * kThreads), x[u]);
    }
  }
  for (; v < nv; v += kThreads) {
    float x[4];
    load4<kGradBf16, kAligned>(s + gs * v, k, x);
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = div(x[j]);
    store4<kOutBf16>(d + os * v, x);
  }
}

template <bool kGradBf16, bool kOutBf16>
__device__ __forceinline__ void rs_tile(const Tile& tl, const PtrArray& grads, uint8_t* __restrict__ rs_in,
                                        DivW div) {
  constexpr uint32_t gsz = kGradBf16 ? 2 : 4;
  constexpr uint32_t osz = kOutBf16 ? 2 : 4;
  {
    uint8_t* d = rs_in + tl.dst * osz;   // 16-byte aligned (tiles start at 16-element offsets)
    const uint32_t n = tl.n;             // multiple of 16
    const uint32_t ns = tl.pad;          // valid source elements
    const uint32_t nv = ns / 4;
    const uint8_t* s = (const uint8_t*)grads.p[tl.param] + tl.src * gsz;
    if (nv > 0) {
      const uint32_t k = (uint32_t)((uintptr_t)s & (kGradBf16 ? 7u : 15u));
      if (k == 0) rs_body<kGradBf16, kOutBf16, true>(s, d, nv, 0, div);
      else rs_body<kGradBf16, kOutBf16, false>(s, d, nv, k, div);
    }
    const uint32_t zb = min((ns + 7u) & ~7u, n);
    for (uint32_t e = nv * 4 + threadIdx.x; e < zb; e += kThreads) {
      float x = 0.0f;
      if (e < ns) {
        if (kGradBf16) x = __uint_as_float(((uint32_t)((const uint16_t*)s)[e]) << 16);
        else x = ((const float*)s)[e];
        x = div(x);
      }
      if (kOutBf16) ((uint16_t*)d)[e] = (uint16_t)(pack_bf16x2(x, 0.0f) & 0xFFFFu);
      else ((float*)d)[e] = x;
    }
    // zero fill [zb, n): padding rows and the alignment gap
    for (uint32_t b = zb * osz + 16 * threadIdx.x; b < n * osz; b += 16 * kThreads)
      st_v4(d + b, make_uint4(0, 0, 0, 0));
  }
}

template <bool kGradBf16, bool kOutBf16>
__global__ void __launch_bounds__(kThreads) k_rs_copy_in(const Tile* __restrict__ tiles, int ntiles,
                                                         PtrArray grads, uint8_t* __restrict__ rs_in,
                                                         DivW div) {
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) rs_tile<kGradBf16, kOutBf16>(tiles[t], grads, rs_in, div);
}

// TMA bulk variant: per 2048-element chunk the TMA engine loads the grad chunk into shared
// memory (mbarrier complete_tx, 2 stages), threads widen / divide / zero-pad into an output
// stage, one thread bulk-stores it (cp.async.bulk shared->global, 2 stages).  Tiles whose
// source is not 16-byte aligned take the register path.
constexpr uint32_t kRsChunk = 2048;

// NS stages (FSDP_B200_K5_STAGES: 2 or 4): chunk i of this CTA uses stage i % NS; the loads
// run NS chunks ahead of the widen / divide and the stores may lag NS - 1 chunks behind.
template <bool kGradBf16, bool kOutBf16, int NS = 2>
__global__ void __launch_bounds__(kThreads) k_rs_copy_in_bulk(const Tile* __restrict__ tiles, int ntiles,
                                                              PtrArray grads, uint8_t* __restrict__ rs_in,
                                                              DivW div) {
  constexpr uint32_t gsz = kGradBf16 ? 2 : 4;
  constexpr uint32_t osz = kOutBf16 ? 2 : 4;
  extern __shared__ __align__(128) uint8_t k5_smem[];   // [NS][chunk * gsz] in, [NS][chunk * osz] out
  uint8_t (*sin)[kRsChunk * gsz] = reinterpret_cast<uint8_t (*)[kRsChunk * gsz]>(k5_smem);
  uint8_t (*sout)[kRsChunk * osz] = reinterpret_cast<uint8_t (*)[kRsChunk * osz]>(k5_smem + NS * kRsChunk * gsz);
  __shared__ uint64_t full[NS];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t it = 0;           // chunks processed by this CTA (stage = it % NS)
  uint32_t loads[NS];        // completed loads per stage barrier (parity = loads & 1)
#pragma unroll
  for (int i = 0; i < NS; ++i) loads[i] = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const uint8_t* s = (const uint8_t*)grads.p[tl.param] + tl.src * gsz;
    uint8_t* d = rs_in + tl.dst * osz;
    const uint32_t n = tl.n, ns = tl.pad;
    if ((((uintptr_t)s) & 15u) != 0 || ((ns * gsz) & 15u) != 0) {
      rs_tile<kGradBf16, kOutBf16>(tl, grads, rs_in, div);
      continue;
    }
    const uint32_t nch = (n + kRsChunk - 1) / kRsChunk;
    auto valid = [&](uint32_t c) -> uint32_t {   // source elements of chunk c
      const uint32_t b = c * kRsChunk;
      const uint32_t ne = min(kRsChunk, n - b);
      return ns > b ? min(ns - b, ne) : 0u;
    };
    auto issue = [&](uint32_t c, uint32_t i) {
      const uint32_t nv = valid(c);
      if (nv == 0) return;
      mbar_arrive_expect_tx(&full[i % NS], nv * gsz);
      bulk_g2s(sin[i % NS], s + (size_t)c * kRsChunk * gsz, nv * gsz, &full[i % NS]);
    };
    if (threadIdx.x == 0) {
      for (uint32_t c = 0; c < (uint32_t)NS && c < nch; ++c) issue(c, it + c);
    }
    for (uint32_t c = 0; c < nch; ++c) {
      const uint32_t i = it + c, st = i % NS;
      const uint32_t ne = min(kRsChunk, n - c * kRsChunk);
      const uint32_t nv = valid(c);
      if (nv > 0) {
        uint32_t par = 0;
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if ((uint32_t)k == st) par = loads[k]++ & 1u;
        mbar_wait(&full[st], par);
      }
      if (threadIdx.x == 0) bulk_wait_read_le<NS - 1>();   // sout[st] (stored NS chunks ago) was read
      __syncthreads();
      for (uint32_t e8 = threadIdx.x; e8 * 8 < ne; e8 += kThreads) {
        float x[8];
        const uint32_t e = e8 * 8;
        if (e + 8 <= nv) {
          if (kGradBf16) {
            const uint4 a = *reinterpret_cast<const uint4*>(sin[st] + e * 2);
            x[0] = bf16_lo(a.x); x[1] = bf16_hi(a.x); x[2] = bf16_lo(a.y); x[3] = bf16_hi(a.y);
            x[4] = bf16_lo(a.z); x[5] = bf16_hi(a.z); x[6] = bf16_lo(a.w); x[7] = bf16_hi(a.w);
          } else {
            const float4 a = *reinterpret_cast<const float4*>(sin[st] + e * 4);
            const float4 b = *reinterpret_cast<const float4*>(sin[st] + e * 4 + 16);
            x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = div(x[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t ej = e + j;
            float v = 0.0f;   // padding rows / alignment gap
            if (ej < nv) {
              v = kGradBf16 ? __uint_as_float(((uint32_t)reinterpret_cast<const uint16_t*>(sin[st])[ej]) << 16)
                            : reinterpret_cast<const float*>(sin[st])[ej];
              v = div(v);
            }
            x[j] = v;
          }
        }
        if (kOutBf16) {
          *reinterpret_cast<uint4*>(sout[st] + e * 2) =
              make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]), pack_bf16x2(x[6], x[7]));
        } else {
          *reinterpret_cast<float4*>(sout[st] + e * 4) = make_float4(x[0], x[1], x[2], x[3]);
          *reinterpret_cast<float4*>(sout[st] + e * 4 + 16) = make_float4(x[4], x[5], x[6], x[7]);
        }
      }
      fence_proxy_async_smem();
      __syncthreads();   // sout[st] complete, sin[st] consumed
      if (threadIdx.x == 0) {
        bulk_s2g(d + (size_t)c * kRsChunk * osz, sout[st], ne * osz);
        bulk_commit();
        if (c + NS < nch) issue(c + NS, i + NS);
      }
    }
    it += nch;
  }
  if (threadIdx.x == 0) bulk_wait0();
}

// ------------------------------------------------------------------- K6 RS copy-out
template <bool kInBf16, bool kAcc>
__global__ void __launch_bounds__(kThreads) k_rs_copy_out(const uint8_t* __restrict__ in,
                                                          float* __restrict__ grad, int64_t n4) {
  // 4 elements per thread per item, so every warp load / store instruction covers one
  // contiguous 256 B (bf16 in) / 512 B span with whole 32 B sectors; kU grid-stride items
  // per thread with all loads issued before any store (HBM latency-bandwidth product)
  constexpr int kU = 4;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  float4* g4 = reinterpret_cast<float4*>(grad);
  for (int64_t base = (int64_t)blockIdx.x * kThreads + threadIdx.x; base < n4; base += kU * stride) {
    uint4 a[kU];
    uint2 h[kU];
    float4 g[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = base + u * stride;
      if (i < n4) {
        if (kInBf16) h[u] = ld_stream8(in + 8 * i);
        else a[u] = ld_stream(in + 16 * i);
        if (kAcc) g[u] = g4[i];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = base + u * stride;
      if (i >= n4) break;
      float4 x;
      if (kInBf16) x = make_float4(bf16_lo(h[u].x), bf16_hi(h[u].x), bf16_lo(h[u].y), bf16_hi(h[u].y));
      else x = make_float4(__uint_as_float(a[u].x), __uint_as_float(a[u].y), __uint_as_float(a[u].z),
                           __uint_as_float(a[u].w));
      if (kAcc) {
        x.x = __fadd_rn(g[u].x, x.x); x.y = __fadd_rn(g[u].y, x.y);
        x.z = __fadd_rn(g[u].z, x.z); x.w = __fadd_rn(g[u].w, x.w);
      }
      g4[i] = x;
    }
  }
}

// ------------------------------------------------------------------- K1 amax
__global__ void __launch_bounds__(kThreads) k_amax(const Tile* __restrict__ tiles, int ntiles,
                                                   uint32_t* __restrict__ acc) {
  __shared__ uint32_t warp_max[kThreads / 32];
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const float* src = reinterpret_cast<const float*>(tl.src);
    const uint32_t n = tl.n;
    const uint32_t nv = n / 4;
    uint32_t m = 0;   // max of |x| bit patterns (non-negative floats order like uints; NaN > inf)
    uint32_t v = threadIdx.x;
    for (; v + (kUnroll - 1) * kThreads < nv; v += kUnroll * kThreads) {
      uint4 q[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) q[u] = ld_stream(src + 4 * (v + u * kThreads));
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        m = max(m, max(max(q[u].x & 0x7FFFFFFFu, q[u].y & 0x7FFFFFFFu),
                       max(q[u].z & 0x7FFFFFFFu, q[u].w & 0x7FFFFFFFu)));
    }
    for (; v < nv; v += kThreads) {
      const uint4 q = ld_stream(src + 4 * v);
      m = max(m, max(max(q.x & 0x7FFFFFFFu, q.y & 0x7FFFFFFFu), max(q.z & 0x7FFFFFFFu, q.w & 0x7FFFFFFFu)));
    }
    for (uint32_t e = nv * 4 + threadIdx.x; e < n; e += kThreads) m = max(m, __float_as_uint(src[e]) & 0x7FFFFFFFu);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0) warp_max[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
      m = threadIdx.x < kThreads / 32 ? warp_max[threadIdx.x] : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
      if (threadIdx.x == 0 && m != 0) atomicMax(acc + tl.param, m);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------- K1b scale
__global__ void k_fp8_scale(const int32_t* __restrict__ idx, int n, uint32_t* __restrict__ acc,
                            float* __restrict__ amax_out, float* __restrict__ scale_out,
                            const uint8_t* __restrict__ eligible, int* __restrict__ err, bool reset) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = idx[i];
  const float a = __uint_as_float(acc[j]);
  amax_out[j] = a;
  float s = 0.0f;
  if (eligible[j]) {
    if (!isfinite(a)) {
      { *(volatile int*)err = 1; __threadfence_system(); }
    } else {
      const float c = fmaxf(a, 1e-12f);
      s = __double2float_rn(__ddiv_rn(448.0, (double)c));
    }
  }
  scale_out[j] = s;
  if (reset) acc[j] = 0u;
}

__global__ void k_fp8_scale_delayed(const int32_t* __restrict__ idx, int n, uint32_t* __restrict__ acc,
                                    float* __restrict__ amax_out, float* __restrict__ scale_out,
                                    const uint8_t* __restrict__ eligible, float* __restrict__ hist,
                                    int32_t* __restrict__ pos, uint8_t* __restrict__ init, int H, int hmax,
                                    int* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = idx[i];
  const float a = __uint_as_float(acc[j]);
  amax_out[j] = a;
  acc[j] = 0u;
  if (!eligible[j]) { scale_out[j] = 0.0f; return; }
  if (!isfinite(a)) { { *(volatile int*)err = 1; __threadfence_system(); } scale_out[j] = 0.0f; return; }
  float* h = hist + (size_t)j * hmax;
  if (!init[j]) {                       // history initialised with the first observed amax
    for (int k = 0; k < H; ++k) h[k] = a;
    pos[j] = 0;
    init[j] = 1;
  }
  float m = h[0];
  for (int k = 1; k < H; ++k) m = fmaxf(m, h[k]);   // max of the history ...
  scale_out[j] = __double2float_rn(__ddiv_rn(448.0, (double)fmaxf(m, 1e-12f)));
  h[pos[j]] = a;                                       // ... updated after use
  pos[j] = pos[j] + 1 == H ? 0 : pos[j] + 1;
}

// K1c: delayed scaling with the amax fused into the casts (kernels.h).  Record, then use.
__global__ void k_fp8_scale_delayed_fused(const int32_t* __restrict__ idx, int n, uint32_t* __restrict__ acc,
                                          float* __restrict__ amax_out, float* __restrict__ scale_out,
                                          const uint8_t* __restrict__ eligible, float* __restrict__ hist,
                                          int32_t* __restrict__ pos, uint8_t* __restrict__ init, int H, int hmax,
                                          int* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = idx[i];
  const float a = __uint_as_float(acc[j]);
  amax_out[j] = a;
  acc[j] = 0u;
  if (!eligible[j]) { scale_out[j] = 0.0f; return; }
  if (!isfinite(a)) { { *(volatile int*)err = 1; __threadfence_system(); } scale_out[j] = 0.0f; return; }
  float* h = hist + (size_t)j * hmax;
  if (!init[j]) {
    for (int k = 0; k < H; ++k) h[k] = a;
    pos[j] = 0;
    init[j] = 1;
  }
  h[pos[j]] = a;                                       // the previous step's amax, recorded ...
  pos[j] = pos[j] + 1 == H ? 0 : pos[j] + 1;
  float m = h[0];
  for (int k = 1; k < H; ++k) m = fmaxf(m, h[k]);      // ... before this step's scale is taken
  scale_out[j] = __double2float_rn(__ddiv_rn(448.0, (double)fmaxf(m, 1e-12f)));
}

inline int grid_for(int64_t work_items, LaunchCfg cfg, int tuned = kCtasCopy) {
  int64_t g = work_items;
  if (g > cfg.cap(tuned)) g = cfg.cap(tuned);
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

cudaError_t launch_copy_in_bf16(const float* shard, void* slot, int64_t S, LaunchCfg cfg, cudaStream_t st) {
  const int64_t n4 = S / 4;
  if (n4 == 0) return cudaSuccess;
  return launch_persistent(k_copy_in_bf16, grid_for((n4 + kThreads - 1) / kThreads, cfg), 0, st,
                           reinterpret_cast<const float4*>(shard), reinterpret_cast<uint2*>(slot), n4);
}

cudaError_t launch_copy_in_fp8(const Tile* tiles, int ntiles, const float* shard, void* slot,
                               const float* scales, LaunchCfg cfg, cudaStream_t st, uint32_t* amax_acc) {
  if (ntiles == 0) return cudaSuccess;
  return launch_persistent(amax_acc ? k_copy_in_fp8<true> : k_copy_in_fp8<false>, grid_for(ntiles, cfg), 0, st,
                           tiles, ntiles, shard, (uint8_t*)slot, scales, amax_acc);
}

cudaError_t launch_copy_out(const Tile* tiles, int ntiles, const void* ag, const PtrArray& outs,
                            LaunchCfg cfg, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  return launch_persistent(k_copy_out, grid_for(ntiles, cfg), 0, st, tiles, ntiles, (const uint8_t*)ag, outs);
}

cudaError_t launch_rs_copy_in(const Tile* tiles, int ntiles, const PtrArray& grads, bool grad_bf16,
                              void* rs_in, bool out_bf16, bool mean, int world_size, LaunchCfg cfg,
                              cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  DivW div;
  div.w = (float)world_size;
  div.pow2 = (world_size & (world_size - 1)) == 0;
  div.inv = 1.0f / (float)world_size;
  div.mean = mean;
  uint8_t* d = (uint8_t*)rs_in;
  if (cfg.variant & 8) {   // TMA bulk K5
    const int gb = grid_for(ntiles, cfg, kCtasCopy);
    const size_t unit = (size_t)kRsChunk * ((grad_bf16 ? 2 : 4) + (out_bf16 ? 2 : 4));
    const int ki = (grad_bf16 ? 2 : 0) + (out_bf16 ? 1 : 0);
    int dev = 0;
    cudaGetDevice(&dev);
    // stages * unit of dynamic shared memory (+ the mbarriers): opt in above the 48 KB default,
    // once per kernel and device
    auto opt_in = [&](auto k, int ns, bool (&done)[4][64]) -> cudaError_t {
      if (dev >= 0 && dev < 64 && done[ki][dev]) return cudaSuccess;
      const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(ns * unit));
      if (e == cudaSuccess && dev >= 0 && dev < 64) done[ki][dev] = true;
      return e;
    };
    if (cfg.k5_stages == 3) {   // the default (FSDP_B200_K5_STAGES): profiles/round2/r2k5
      auto k = grad_bf16 ? (out_bf16 ? k_rs_copy_in_bulk<true, true, 3> : k_rs_copy_in_bulk<true, false, 3>)
                         : (out_bf16 ? k_rs_copy_in_bulk<false, true, 3> : k_rs_copy_in_bulk<false, false, 3>);
      static bool attr3[4][64] = {};
      const cudaError_t e = opt_in(k, 3, attr3);
      if (e != cudaSuccess) return e;
      return launch_persistent(k, gb, 3 * unit, st, tiles, ntiles, grads, d, div);
    }
    if (cfg.k5_stages == 4) {
      auto k = grad_bf16 ? (out_bf16 ? k_rs_copy_in_bulk<true, true, 4> : k_rs_copy_in_bulk<true, false, 4>)
                         : (out_bf16 ? k_rs_copy_in_bulk<false, true, 4> : k_rs_copy_in_bulk<false, false, 4>);
      static bool attr4[4][64] = {};
      const cudaError_t e = opt_in(k, 4, attr4);
      if (e != cudaSuccess) return e;
      return launch_persistent(k, gb, 4 * unit, st, tiles, ntiles, grads, d, div);
    }
    auto k = grad_bf16 ? (out_bf16 ? k_rs_copy_in_bulk<true, true> : k_rs_copy_in_bulk<true, false>)
                       : (out_bf16 ? k_rs_copy_in_bulk<false, true> : k_rs_copy_in_bulk<false, false>);
    return launch_persistent(k, gb, 2 * unit, st, tiles, ntiles, grads, d, div);
  }
  const int g = grid_for(ntiles, cfg, kCtasRsCopyIn);
  auto k = grad_bf16 ? (out_bf16 ? k_rs_copy_in<true, true> : k_rs_copy_in<true, false>)
                     : (out_bf16 ? k_rs_copy_in<false, true> : k_rs_copy_in<false, false>);
  return launch_persistent(k, g, 0, st, tiles, ntiles, grads, d, div);
}

cudaError_t launch_rs_copy_out(const void* rs_out, bool in_bf16, float* grad, bool accumulate, int64_t S,
                               LaunchCfg cfg, cudaStream_t st) {
  const int64_t n4 = S / 4;   // S is a multiple of 16 (R2)
  if (n4 == 0) return cudaSuccess;
  const int g = grid_for((n4 + kThreads - 1) / kThreads, cfg);
  const uint8_t* in = (const uint8_t*)rs_out;
  auto k = in_bf16 ? (accumulate ? k_rs_copy_out<true, true> : k_rs_copy_out<true, false>)
                   : (accumulate ? k_rs_copy_out<false, true> : k_rs_copy_out<false, false>);
  return launch_persistent(k, g, 0, st, in, grad, n4);
}

cudaError_t launch_amax(const Tile* tiles, int ntiles, uint32_t* acc_bits, LaunchCfg cfg, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  return launch_persistent(k_amax, grid_for(ntiles, cfg), 0, st, tiles, ntiles, acc_bits);
}

cudaError_t launch_fp8_scale(const int32_t* idx, int n, uint32_t* acc_bits, float* amax_out, float* scale_out,
                             const uint8_t* eligible, int* err_flag, bool reset_acc, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_fp8_scale<<<(n + 127) / 128, 128, 0, st>>>(idx, n, acc_bits, amax_out, scale_out, eligible, err_flag,
                                                 reset_acc);
  return cudaGetLastError();
}

}  // namespace fsdpk

namespace fsdpk {
cudaError_t launch_fp8_scale_delayed(const int32_t* idx, int n, uint32_t* acc_bits, float* amax_out, float* scale_out,
                                     const uint8_t* eligible, float* hist, int32_t* pos, uint8_t* hist_init, int H,
                                     int hmax, int* err_flag, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_fp8_scale_delayed<<<(n + 127) / 128, 128, 0, st>>>(idx, n, acc_bits, amax_out, scale_out, eligible, hist, pos,
                                                         hist_init, H, hmax, err_flag);
  return cudaGetLastError();
}

cudaError_t launch_fp8_scale_delayed_fused(const int32_t* idx, int n, uint32_t* acc_bits, float* amax_out,
                                           float* scale_out, const uint8_t* eligible, float* hist, int32_t* pos,
                                           uint8_t* hist_init, int H, int hmax, int* err_flag, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_fp8_scale_delayed_fused<<<(n + 127) / 128, 128, 0, st>>>(idx, n, acc_bits, amax_out, scale_out, eligible, hist,
                                                               pos, hist_init, H, hmax, err_flag);
  return cudaGetLastError();
}
}  // namespace fsdpk

namespace fsdpdev {
int resident_ctas(const void* fn, size_t dyn_smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, size_t, int>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const auto key = std::make_tuple(fn, dyn_smem, dev);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, dyn_smem) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;   // unknown: the caller keeps its grid
  }
  const int r = per_sm * sms;
  cache[key] = r;
  return r;
}
}  // namespace fsdpdev
