// umma_probe.cu — microbenchmark: throughput of back-to-back tcgen05.mma kind::f16 (M = 128, K = 16)
// on one CTA per SM, A from TMEM (TS) or from shared memory (SS), for N = 16 .. 256.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include -I../paper_2308_09723_b200/csrc
//        umma_probe.cu -o umma_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "fq_common.cuh"
#include "fq_tcgen05.cuh"

using namespace fq;
using namespace fq::tc5;

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16<__half, 128, N>();
    const uint32_t b_addr = smem_u32(base) + 128 * 128;
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const uint64_t bdesc = sw128_desc(b_addr) + (uint64_t)((kk % 4) * 2);
        if (TS) {
          mma_ts(tm + 256, tm + (kk % 8) * 8 + (kk / 8) * 64, bdesc, idesc, kk != 0);
        } else {
          const uint64_t adesc = sw128_desc(smem_u32(base)) + (uint64_t)((kk % 4) * 2);
          mma_ss(tm + 256, adesc, bdesc, idesc, kk != 0);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    tmem_dealloc(tm, 512);
  }
}

// Same loop without waiting for each commit (up to 16 x 16 MMAs in flight)
template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe_stream(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ uint32_t tbase;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16<__half, 128, N>();
    const uint32_t b_addr = smem_u32(base) + 128 * 128;
    const long long t0 = clock64();
    uint32_t ph[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
      const int b = it & 3;
      if (it >= 4) {
        mbar_wait(&bar[b], ph[b]);
        ph[b] ^= 1;
      }
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const uint64_t bdesc = sw128_desc(b_addr) + (uint64_t)((kk % 4) * 2);
        if (TS) {
          mma_ts(tm + 256 + (N <= 128 ? (b & 1) * N : 0), tm + (kk % 8) * 8 + (kk / 8) * 64, bdesc, idesc, kk != 0);
        } else {
          const uint64_t adesc = sw128_desc(smem_u32(base)) + (uint64_t)((kk % 4) * 2);
          mma_ss(tm + 256 + (N <= 128 ? (b & 1) * N : 0), adesc, bdesc, idesc, kk != 0);
        }
      }
      mma_commit(&bar[b]);
    }
    for (int b = 0; b < 4; ++b) mbar_wait(&bar[b], ph[b]);
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <int N, bool TS, bool STREAM>
void run(long long* d, long long* h, int nsm) {
  const int iters = 2000;
  auto k = STREAM ? probe_stream<N, TS> : probe<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<nsm, 128, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d %s: %s\n", N, TS ? "TS" : "SS", cudaGetErrorString(e));
    return;
  }
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double per = avg / (iters * 16.0);
  printf("%s %s N=%3d: %7.1f cycles per MMA (M=128 K=16), %6.1f B/cycle of A, %7.1f MAC/cycle\n",
         STREAM ? "stream" : "commit-wait", TS ? "TS" : "SS", N, per, 4096.0 / per, 128.0 * N * 16 / per);
}

// cta_group::2 (CTA pair, M = 256): only the leader issues; A rows and B columns are split over
// the pair (each CTA's smem holds 128 rows of A and N/2 rows of B); commit multicast to both CTAs.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe_pair(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  fence_proxy_async_smem();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  fence_after();
  const uint32_t tm = tbase;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16<__half, 256, N>();
    const uint32_t b_addr = smem_u32(base) + 128 * 128;
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const uint64_t bdesc = sw128_desc(b_addr) + (uint64_t)((kk % 4) * 2);
        const uint64_t adesc = sw128_desc(smem_u32(base)) + (uint64_t)((kk % 4) * 2);
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + 256),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)(kk != 0)));
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    const long long t1 = clock64();
    cycles[blockIdx.x / 2] = t1 - t0;
  }
  fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
  }
}

template <int N>
void run_pair(long long* d, long long* h, int nsm) {
  const int iters = 2000;
  cudaFuncSetAttribute(probe_pair<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  probe_pair<N><<<nsm, 128, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("pair N=%d: %s\n", N, cudaGetErrorString(e));
    return;
  }
  cudaMemcpy(h, d, nsm / 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm / 2; ++i) avg += h[i];
  avg /= nsm / 2;
  const double per = avg / (iters * 16.0);
  printf("pair SS M=256 N=%3d: %7.1f cycles per MMA, %6.1f weights (M x K) per cycle per SM\n", N, per,
         128.0 * 16 / per);
}

template <int N>
__global__ void __launch_bounds__(128, 1) probe_m64(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16<__half, 64, N>();
    const uint32_t b_addr = smem_u32(base) + 128 * 128;
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const uint64_t bdesc = sw128_desc(b_addr) + (uint64_t)((kk % 4) * 2);
        const uint64_t adesc = sw128_desc(smem_u32(base)) + (uint64_t)((kk % 4) * 2);
        mma_ss(tm + 256, adesc, bdesc, idesc, kk != 0);
      }
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <int N>
void run_m64(long long* d, long long* h, int nsm) {
  const int iters = 2000;
  cudaFuncSetAttribute(probe_m64<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  probe_m64<N><<<nsm, 128, 100 * 1024>>>(iters, d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("m64 failed\n"); return; }
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double per = avg / (iters * 16.0);
  printf("SS M=64 N=%3d: %7.1f cycles per MMA, %6.1f weights (M x K) per cycle per SM\n", N, per, 64.0 * 16 / per);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *d, h[1024];
  cudaMalloc(&d, 1024 * sizeof(long long));
  run<16, true, false>(d, h, nsm);
  run<16, true, true>(d, h, nsm);
  run<32, true, true>(d, h, nsm);
  run<64, true, true>(d, h, nsm);
  run<128, true, true>(d, h, nsm);
  run<256, true, true>(d, h, nsm);
  run<16, false, true>(d, h, nsm);
  run<32, false, true>(d, h, nsm);
  run<64, false, true>(d, h, nsm);
  run<128, false, true>(d, h, nsm);
  run<256, false, true>(d, h, nsm);
  run<64, false, false>(d, h, nsm);
  run_m64<64>(d, h, nsm);
  run_m64<16>(d, h, nsm);
  run_pair<32>(d, h, nsm);
  run_pair<64>(d, h, nsm);
  run_pair<128>(d, h, nsm);
  run_pair<256>(d, h, nsm);
  return 0;
}
