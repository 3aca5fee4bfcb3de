// Device helpers shared by the segmented copy kernels (kernels.cu) and the fused
// peer-memory kernels (p2p_kernels.cu).  Internal; header-only.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fsdpdev {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// fp32 pair -> packed bf16x2, round to nearest even (cvt.rn.bf16x2.f32; lo in low half).
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// fp32 pair -> packed e4m3x2 with saturation to +-448 (cvt.rn.satfinite; lo in low byte).
__device__ __forceinline__ uint32_t pack_e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return (uint32_t)r;
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// 16 bytes starting at byte phase k (1..15) of the 32 bytes a:b.
__device__ __forceinline__ uint4 extract16(uint4 a, uint4 b, uint32_t k) {
  const uint32_t sh = (k & 3u) * 8u;
  uint4 r;
  switch (k >> 2) {
    case 0:
      r.x = __funnelshift_r(a.x, a.y, sh); r.y = __funnelshift_r(a.y, a.z, sh);
      r.z = __funnelshift_r(a.z, a.w, sh); r.w = __funnelshift_r(a.w, b.x, sh);
      break;
    case 1:
      r.x = __funnelshift_r(a.y, a.z, sh); r.y = __funnelshift_r(a.z, a.w, sh);
      r.z = __funnelshift_r(a.w, b.x, sh); r.w = __funnelshift_r(b.x, b.y, sh);
      break;
    case 2:
      r.x = __funnelshift_r(a.z, a.w, sh); r.y = __funnelshift_r(a.w, b.x, sh);
      r.z = __funnelshift_r(b.x, b.y, sh); r.w = __funnelshift_r(b.y, b.z, sh);
      break;
    default:
      r.x = __funnelshift_r(a.w, b.x, sh); r.y = __funnelshift_r(b.x, b.y, sh);
      r.z = __funnelshift_r(b.y, b.z, sh); r.w = __funnelshift_r(b.z, b.w, sh);
      break;
  }
  return r;
}

// 16 bytes at an arbitrary address whose phase within 16 B is `k` (uniform per tile).
// For k != 0 two aligned loads are made; the second aligned block always contains at
// least one requested byte, so it lies inside the (>= 16 B granular) allocation.
template <bool kAligned>
__device__ __forceinline__ uint4 load16(const uint8_t* p, uint32_t k) {
  if (kAligned) return ld_stream(p);
  const uint8_t* a = p - k;
  return extract16(ld_stream(a), ld_stream(a + 16), k);
}

template <bool kAligned>
__device__ __forceinline__ void copy_body(const uint8_t* s, uint8_t* d, uint32_t nv, uint32_t k) {
  uint32_t v = threadIdx.x;
  for (; v + (kUnroll - 1) * kThreads < nv; v += kUnroll * kThreads) {
    uint4 r[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) r[u] = load16<kAligned>(s + 16 * (v + u * kThreads), k);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_v4(d + 16 * (v + u * kThreads), r[u]);
  }
  for (; v < nv; v += kThreads) st_v4(d + 16 * v, load16<kAligned>(s + 16 * v, k));
}


}  // namespace fsdpdev
