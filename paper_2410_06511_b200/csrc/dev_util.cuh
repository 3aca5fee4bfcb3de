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


__device__ __forceinline__ void st_v2(void* p, uint2 v) {
  asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}

__device__ __forceinline__ uint2 ld_stream8(const void* p) {
  uint2 a;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(a.x), "=r"(a.y) : "l"(p));
  return a;
}

// ---- TMA bulk copies (cp.async.bulk) + mbarrier, sm_90+/sm_100a (SASS UBLKCP)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global (local or peer-mapped) -> shared, completes `bytes` on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global (local or peer-mapped), tracked by the bulk async-group of this thread
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_le1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
template <int N>   // at most N bulk store groups still reading shared memory
__device__ __forceinline__ void bulk_wait_read_le() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// L1-allocating variants for the misaligned phase of peer (NVLink) reads: the two aligned
// blocks a lane loads overlap its neighbour's, and peer data bypasses L2 (cached in L1
// only), so without L1 allocation every remote byte would cross NVLink twice.
__device__ __forceinline__ uint2 ld_l1_8(const void* p) {
  uint2 a;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(a.x), "=r"(a.y) : "l"(p));
  return a;
}
__device__ __forceinline__ uint4 ld_l1_16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// 4 consecutive peer grad elements (as fp32), misaligned phase k != 0, L1-allocating loads.
template <bool kGradBf16>
__device__ __forceinline__ void load4_peer_misaligned(const uint8_t* p, uint32_t k, float (&x)[4]) {
  if (kGradBf16) {
    const uint8_t* b = p - k;
    const uint2 u = ld_l1_8(b), w = ld_l1_8(b + 8);
    const uint32_t sh = (k & 3u) * 8u;
    uint2 a;
    if (k < 4) { a.x = __funnelshift_r(u.x, u.y, sh); a.y = __funnelshift_r(u.y, w.x, sh); }
    else { a.x = __funnelshift_r(u.y, w.x, sh); a.y = __funnelshift_r(w.x, w.y, sh); }
    x[0] = bf16_lo(a.x); x[1] = bf16_hi(a.x); x[2] = bf16_lo(a.y); x[3] = bf16_hi(a.y);
  } else {
    const uint8_t* b = p - k;
    const uint4 a = extract16(ld_l1_16(b), ld_l1_16(b + 16), k);
    x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y);
    x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
  }
}

// 4 consecutive grad elements (as fp32) at byte address p whose phase is k: bf16 grads are
// read as one 8-byte load (k in {0,2,4,6}: two aligned loads + funnel shift when k != 0),
// fp32 grads as one 16-byte load (k in {0,4,8,12}).
template <bool kGradBf16, bool kAligned>
__device__ __forceinline__ void load4(const uint8_t* p, uint32_t k, float (&x)[4]) {
  if (kGradBf16) {
    uint2 a;
    if (kAligned) {
      a = ld_stream8(p);
    } else {
      const uint8_t* b = p - k;
      const uint2 u = ld_stream8(b), w = ld_stream8(b + 8);
      const uint32_t sh = (k & 3u) * 8u;
      if (k < 4) { a.x = __funnelshift_r(u.x, u.y, sh); a.y = __funnelshift_r(u.y, w.x, sh); }
      else { a.x = __funnelshift_r(u.y, w.x, sh); a.y = __funnelshift_r(w.x, w.y, sh); }
    }
    x[0] = bf16_lo(a.x); x[1] = bf16_hi(a.x); x[2] = bf16_lo(a.y); x[3] = bf16_hi(a.y);
  } else {
    const uint4 a = load16<kAligned>(p, k);
    x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y);
    x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
  }
}

// Programmatic dependent launch: a kernel launched with programmatic stream serialization
// may start while its predecessor on the stream is still running; it must call this first,
// which waits until the predecessor grid completed and its memory is visible.  A no-op for
// kernels launched normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- host: persistent-grid launches
// CTAs of `fn` (kThreads threads, `dyn_smem` dynamic bytes, plus its registers and static
// shared memory) the whole GPU holds at once; cached per kernel (kernels.cu).
int resident_ctas(const void* fn, size_t dyn_smem);

// Launches a persistent tile-loop kernel with min(g, resident CTAs) CTAs: a CTA that does
// not fit in the first wave would start only after a first-wave CTA finished ALL of its
// tiles, so an oversized grid turns into a tail of serial work.
template <class... KArgs, class... Args>
cudaError_t launch_persistent(void (*kern)(KArgs...), int g, size_t dyn_smem, cudaStream_t st, Args&&... args) {
  const int r = resident_ctas(reinterpret_cast<const void*>(kern), dyn_smem);
  if (r > 0 && g > r) g = r;
  if (g < 1) g = 1;
  kern<<<g, kThreads, dyn_smem, st>>>(static_cast<Args&&>(args)...);
  return cudaGetLastError();
}

// Launch with programmatic stream serialization (the kernel must start with pdl_wait()):
// its launch latency overlaps the tail of the previous kernel on `st`.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), int g, int threads, size_t dyn_smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3((unsigned)g);
  c.blockDim = dim3((unsigned)threads);
  c.dynamicSmemBytes = dyn_smem;
  c.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = a;
  c.numAttrs = 1;
  return cudaLaunchKernelEx(&c, kern, static_cast<Args&&>(args)...);
}

// launch_persistent's grid sizing with a programmatic-dependent launch
template <class... KArgs, class... Args>
cudaError_t launch_persistent_pdl(void (*kern)(KArgs...), int g, size_t dyn_smem, cudaStream_t st, Args&&... args) {
  const int r = resident_ctas(reinterpret_cast<const void*>(kern), dyn_smem);
  if (r > 0 && g > r) g = r;
  if (g < 1) g = 1;
  return launch_pdl(kern, g, kThreads, dyn_smem, st, static_cast<Args&&>(args)...);
}

}  // namespace fsdpdev
