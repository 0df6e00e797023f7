// umma_probe2.cu — microbenchmark: does the per-instruction cost of small-N tcgen05.mma come from
// the accumulator dependency chain?  Back-to-back MMAs (M = 128) rotating over NACC independent
// TMEM accumulators, kind::f16 (K = 16) and kind::i8 (K = 32), A from shared memory (SS) or TMEM (TS).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include
//        -I../paper_2308_09723_b200/csrc umma_probe2.cu -o umma_probe2
#include <cstdio>
#include <cuda_runtime.h>

#include "fq_common.cuh"
#include "fq_tcgen05.cuh"

using namespace fq;
using namespace fq::tc5;

template <bool I8, bool TS>
__device__ __forceinline__ void mma(uint32_t d, uint64_t adesc, uint32_t atm, uint64_t bdesc, uint32_t idesc,
                                    uint32_t acc) {
  if (I8) {
    if (TS)
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                   "r"(atm), "l"(bdesc), "r"(idesc), "r"(acc));
    else
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                   "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  } else {
    if (TS)
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                   "r"(atm), "l"(bdesc), "r"(idesc), "r"(acc));
    else
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                   "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  }
}

template <bool I8, int N>
__host__ __device__ constexpr uint32_t idesc_of() {
  return I8 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24))
            : idesc_f16<__half, 128, N>();
}

// NACC accumulators at TMEM columns 256 + a * N (a < NACC); A (TS) at columns 0..63.
template <bool I8, bool TS, int N, int NACC>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* cycles) {
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
    constexpr uint32_t idesc = idesc_of<I8, N>();
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
        const uint64_t adesc = sw128_desc(smem_u32(base)) + (uint64_t)((kk % 4) * 2);
        const uint32_t d = tm + 256 + (kk % NACC) * N;
        mma<I8, TS>(d, adesc, tm + (kk % 8) * 8, bdesc, idesc, it != 0 || kk >= NACC);
      }
      mma_commit(&bar[b]);
    }
    for (int b = 0; b < 4; ++b) mbar_wait(&bar[b], ph[b]);
    cycles[blockIdx.x] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <bool I8, bool TS, int N, int NACC>
void run(long long* d, long long* h, int nsm) {
  static_assert(NACC * N <= 256, "accumulators fit");
  const int iters = 2000;
  auto k = probe<I8, TS, N, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<nsm, 128, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s %s N=%d NACC=%d: %s\n", I8 ? "i8 " : "f16", TS ? "TS" : "SS", N, NACC, cudaGetErrorString(e));
    return;
  }
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double per = avg / (iters * 16.0);
  const int K = I8 ? 32 : 16;
  printf("%s %s N=%3d NACC=%d: %6.1f cycles per MMA (M=128 K=%d): %6.1f weights/cycle/SM\n", I8 ? "i8 " : "f16",
         TS ? "TS" : "SS", N, NACC, per, K, 128.0 * K / per);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *d, h[1024];
  cudaMalloc(&d, 1024 * sizeof(long long));
  run<false, false, 16, 1>(d, h, nsm);
  run<false, false, 16, 4>(d, h, nsm);
  run<false, false, 16, 8>(d, h, nsm);
  run<false, true, 16, 1>(d, h, nsm);
  run<false, true, 16, 8>(d, h, nsm);
  run<false, false, 32, 8>(d, h, nsm);
  run<false, false, 64, 4>(d, h, nsm);
  run<true, false, 16, 1>(d, h, nsm);
  run<true, false, 16, 4>(d, h, nsm);
  run<true, false, 16, 8>(d, h, nsm);
  run<true, true, 16, 1>(d, h, nsm);
  run<true, true, 16, 8>(d, h, nsm);
  run<true, false, 32, 1>(d, h, nsm);
  run<true, false, 32, 8>(d, h, nsm);
  run<true, true, 32, 8>(d, h, nsm);
  run<true, false, 64, 4>(d, h, nsm);
  run<true, true, 64, 4>(d, h, nsm);
  run<true, false, 128, 2>(d, h, nsm);
  run<true, false, 256, 1>(d, h, nsm);
  run<false, false, 256, 1>(d, h, nsm);
  return 0;
}
