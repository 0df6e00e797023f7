// hmma_probe.cu — legacy tensor-core throughput on sm_100a: mma.sync.m16n8k16 (f16 -> f32) per SM
// with W warps per CTA (1 CTA per SM) and C independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int C>
__global__ void hmma(int iters, float* out, long long* cyc) {
  float acc[C][4];
  for (int c = 0; c < C; ++c) for (int i = 0; i < 4; ++i) acc[c][i] = 0.f;
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3, threadIdx.x * 5, threadIdx.x * 7};
  uint32_t b0 = threadIdx.x * 11, b1 = threadIdx.x * 13;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < C; ++c) for (int i = 0; i < 4; ++i) s += acc[c][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps, int nsm, float* o, long long* d) {
  const int iters = 4096;
  hmma<C><<<nsm, 32 * warps>>>(iters, o, d);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  const double per_sm = (double)iters * C * warps / avg;  // HMMA per cycle per SM
  printf("warps=%2d chains=%d: %.3f HMMA.16816/cycle/SM = %.0f TFLOP/s at 1.965 GHz x %d SMs\n", warps, C, per_sm,
         per_sm * 4096 * 1.965e9 * nsm / 1e12, nsm);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  long long* d;
  cudaMalloc(&o, nsm * 1024 * 4);
  cudaMalloc(&d, 1024 * 8);
  for (int w : {4, 8, 16, 32}) {
    run<1>(w, nsm, o, d);
    run<2>(w, nsm, o, d);
    run<4>(w, nsm, o, d);
  }
  return 0;
}
