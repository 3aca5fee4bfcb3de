// NVLink ceiling probe (2 GPUs, one process): what each transfer mechanism reaches between
// two B200s through NVSwitch, one-way and in both directions at once (the fused push / pull
// kernels move data both ways simultaneously).  Mechanisms:
//   ce      cudaMemcpyPeerAsync (copy engines)
//   st      SM kernel, 16-byte stores to the peer (the register push path)
//   ld      SM kernel, 16-byte loads from the peer, stored locally (the register pull path)
//   tma_ld  SM kernel, cp.async.bulk global->shared from the peer (the bulk pull path)
//   tma_st  SM kernel, cp.async.bulk shared->global to the peer (the bulk push path)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe scripts/nvlink_probe.cu
// Run:   ./nvlink_probe [MiB per direction, default 1024]   -> one JSON line per test
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

constexpr int kThreads = 256;

__global__ void k_store(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kThreads)
    dst[i] = src[i];
}

__global__ void k_load(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  constexpr int U = 4;
  const size_t stride = (size_t)gridDim.x * kThreads;
  for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) dst[i + u * stride] = v[u];
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// cp.async.bulk peer -> smem (4 KB chunks, 2 stages, mbarrier), then smem -> local global
__global__ void k_tma_load(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t bytes) {
  constexpr uint32_t C = 4096;
  __shared__ __align__(128) uint8_t buf[2][C];
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nch = bytes / C;
  auto issue = [&](size_t c, uint32_t s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(C));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(buf[s])),
                 "l"(src + c * C), "r"(C), "r"(smem_u32(&bar[s]))
                 : "memory");
  };
  uint32_t k = 0;
  size_t c = blockIdx.x;
  if (threadIdx.x == 0) {
    if (c < nch) issue(c, 0);
    if (c + gridDim.x < nch) issue(c + gridDim.x, 1);
  }
  for (; c < nch; c += gridDim.x, ++k) {
    const uint32_t s = k & 1u, par = (k >> 1) & 1u;
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
            smem_u32(&bar[s])),
        "r"(par)
        : "memory");
    reinterpret_cast<uint4*>(dst + c * C)[threadIdx.x] = reinterpret_cast<const uint4*>(buf[s])[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && c + 2 * (size_t)gridDim.x < nch) issue(c + 2 * (size_t)gridDim.x, s);
  }
}

// local global -> smem (plain loads), then cp.async.bulk smem -> peer (4 KB chunks, 2 stages)
__global__ void k_tma_store(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t bytes) {
  constexpr uint32_t C = 4096;
  __shared__ __align__(128) uint8_t buf[2][C];
  const size_t nch = bytes / C;
  uint32_t k = 0;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x, ++k) {
    const uint32_t s = k & 1u;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    reinterpret_cast<uint4*>(buf[s])[threadIdx.x] = reinterpret_cast<const uint4*>(src + c * C)[threadIdx.x];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * C),
                   "r"(smem_u32(buf[s])), "r"(C)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const size_t mib = argc > 1 ? strtoull(argv[1], nullptr, 10) : 1024;
  const size_t bytes = mib << 20;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("{\"error\": \"need 2 GPUs\"}\n");
    return 0;
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t *a[2], *b[2];   // a[d]: source on device d; b[d]: destination on device d
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], d + 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  const char* names[] = {"ce", "st", "ld", "tma_ld", "tma_st"};
  for (int m = 0; m < 5; ++m) {
    for (int bidir = 0; bidir < 2; ++bidir) {
      for (int grid_mult : {1, 2, 4, 8}) {
        if (m == 0 && grid_mult > 1) continue;
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaDeviceSynchronize());
          }
          for (int d = 0; d < 1 + bidir; ++d) {
            // transfer d -> 1-d, issued by device d (push mechanisms) or 1-d (pull mechanisms)
            const bool pull = (m == 2 || m == 3);
            const int issuer = pull ? 1 - d : d;   // streams / events belong to the issuing device
            CK(cudaSetDevice(issuer));
            CK(cudaEventRecord(e0[issuer], st[issuer]));
            const int g = sms * grid_mult;
            cudaStream_t s = st[issuer];
            if (m == 0) CK(cudaMemcpyPeerAsync(b[1 - d], 1 - d, a[d], d, bytes, s));
            else if (m == 1) k_store<<<g, kThreads, 0, s>>>((const uint4*)a[d], (uint4*)b[1 - d], bytes / 16);
            else if (m == 2) k_load<<<g, kThreads, 0, s>>>((const uint4*)a[d], (uint4*)b[1 - d], bytes / 16);
            else if (m == 3) k_tma_load<<<g, kThreads, 0, s>>>(a[d], b[1 - d], bytes);
            else k_tma_store<<<g, kThreads, 0, s>>>(a[d], b[1 - d], bytes);
            CK(cudaGetLastError());
            CK(cudaEventRecord(e1[issuer], st[issuer]));
          }
          float worst = 0.f;
          for (int d = 0; d < 1 + bidir; ++d) {
            const int issuer = (m == 2 || m == 3) ? 1 - d : d;
            CK(cudaSetDevice(issuer));
            CK(cudaEventSynchronize(e1[issuer]));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0[issuer], e1[issuer]));
            if (ms > worst) worst = ms;
          }
          if (rep > 0 && worst < best) best = worst;
        }
        printf("{\"mech\": \"%s\", \"bidirectional\": %s, \"ctas_per_sm\": %d, \"MiB\": %zu, \"ms\": %.4f, "
               "\"GBps_per_direction\": %.1f}\n",
               names[m], bidir ? "true" : "false", m == 0 ? 0 : grid_mult, mib, best, bytes / (best * 1e-3) / 1e9);
        fflush(stdout);
      }
    }
  }
  // all-to-all over every visible GPU (the unshard / reduce-scatter pattern): each device
  // sends bytes/(N-1) to every peer at once; copy engines (one stream per peer) vs one SM
  // store kernel per peer (each with sms*4/(N-1) CTAs) vs SM loads (each device pulls)
  if (ndev > 2) {
    const int N = ndev;
    for (int d = 2; d < N; ++d) {
      CK(cudaSetDevice(d));
      for (int q = 0; q < N; ++q)
        if (q != d) cudaDeviceEnablePeerAccess(q, 0);
    }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      for (int q = 2; q < N; ++q) cudaDeviceEnablePeerAccess(q, 0);
    }
    cudaGetLastError();
    uint8_t* src[8];
    uint8_t* dst[8];
    cudaStream_t ss[8][8];
    cudaEvent_t f0[8], f1[8];
    const size_t part = (bytes / (N - 1)) & ~(size_t)4095;
    for (int d = 0; d < N; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMalloc(&src[d], part * N));
      CK(cudaMalloc(&dst[d], part * N));
      CK(cudaMemset(src[d], d + 1, part * N));
      for (int q = 0; q < N; ++q) CK(cudaStreamCreateWithFlags(&ss[d][q], cudaStreamNonBlocking));
      CK(cudaEventCreate(&f0[d]));
      CK(cudaEventCreate(&f1[d]));
    }
    const char* an[] = {"a2a_ce", "a2a_st", "a2a_ld", "a2a_ce_plus_st"};
    for (int m = 0; m < 4; ++m) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaDeviceSynchronize());
        }
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(f0[d], ss[d][d]));
          for (int q = 0; q < N; ++q)
            if (q != d) CK(cudaStreamWaitEvent(ss[d][q], f0[d], 0));
          for (int q = 0; q < N; ++q) {
            if (q == d) continue;
            const int g = sms * 4 / (N - 1);
            // d's piece for q: src[d] + q*part -> dst[q] + d*part (push), or pulled by d from q
            if (m == 0) CK(cudaMemcpyPeerAsync(dst[q] + d * part, q, src[d] + q * part, d, part, ss[d][q]));
            else if (m == 1) k_store<<<g, kThreads, 0, ss[d][q]>>>((const uint4*)(src[d] + q * part),
                                                                  (uint4*)(dst[q] + d * part), part / 16);
            else if (m == 2) k_load<<<g, kThreads, 0, ss[d][q]>>>((const uint4*)(src[q] + d * part),
                                                                 (uint4*)(dst[d] + q * part), part / 16);
            else {   // half of each peer's bytes by copy engine, half by SM stores, concurrently
              const size_t h = (part / 2) & ~(size_t)4095;
              CK(cudaMemcpyPeerAsync(dst[q] + d * part, q, src[d] + q * part, d, h, ss[d][q]));
              k_store<<<g, kThreads, 0, ss[d][(q + 1) % N == d ? (q + 2) % N : (q + 1) % N]>>>(
                  (const uint4*)(src[d] + q * part + h), (uint4*)(dst[q] + d * part + h), (part - h) / 16);
            }
            CK(cudaGetLastError());
          }
          for (int q = 0; q < N; ++q) {
            if (q == d) continue;
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, ss[d][q]));
            CK(cudaStreamWaitEvent(ss[d][d], e, 0));
            CK(cudaEventDestroy(e));
          }
          CK(cudaEventRecord(f1[d], ss[d][d]));
        }
        float worst = 0.f;
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(f1[d]));
          float ms = 0.f;
          CK(cudaEventElapsedTime(&ms, f0[d], f1[d]));
          if (ms > worst) worst = ms;
        }
        if (rep > 0 && worst < best) best = worst;
      }
      printf("{\"mech\": \"%s\", \"gpus\": %d, \"MiB_per_gpu_each_direction\": %.1f, \"ms\": %.4f, "
             "\"GBps_per_direction\": %.1f}\n",
             an[m], N, part * (N - 1) / 1048576.0, best, part * (N - 1) / (best * 1e-3) / 1e9);
      fflush(stdout);
    }
  }
  return 0;
}
