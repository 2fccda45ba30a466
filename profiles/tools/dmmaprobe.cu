#include <cstdio>
#include <cuda_runtime.h>
// Does the FP64 tensor path (DMMA, mma.sync m8n8k4 f64) issue beside the
// FP64 FMA pipe? MODE 0: every warp DFMA; 1: every warp DMMA; 2: even warps
// DFMA, odd warps DMMA (aggregate > either alone => separate pipes).
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void __launch_bounds__(256) probe(double* out, int iters, double a, double b, long long* cnt) {
  const int warp = threadIdx.x >> 5;
  const bool tc = MODE == 1 || (MODE == 2 && (warp & 1));
  double s = 0;
  if (tc) {
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma(c[k], a, b);
    }
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (threadIdx.x % 32 == 0) atomicAdd((unsigned long long*)cnt, (unsigned long long)iters * 8 * 512);
  } else {
    double x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = fma(x[k], a, b);
    }
    for (int i = 0; i < 16; ++i) s += x[i];
    if (threadIdx.x % 32 == 0) atomicAdd((unsigned long long*)cnt + 1, (unsigned long long)iters * 16 * 64);
  }
  if (s == 12345.6789) out[0] = s;
}
template <int M> void run(int sms, int bps, int iters_tc, int iters_fma) {
  double* d; cudaMalloc(&d, 8);
  long long* cnt; cudaMalloc(&cnt, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * bps;
  int iters = M == 1 ? iters_tc : iters_fma;
  probe<M><<<blocks, 256>>>(d, 4, 0.999999, 1e-7, cnt);
  cudaMemset(cnt, 0, 16);
  cudaEventRecord(e0);
  probe<M><<<blocks, 256>>>(d, iters, 0.999999, 1e-7, cnt);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[2]; cudaMemcpy(h, cnt, 16, cudaMemcpyDeviceToHost);
  printf("mode %d blocks/SM %d: %.3f ms, DMMA %.1f TF, DFMA %.1f TF, total %.1f TF (%s)\n", M, bps, ms,
         h[0] / (ms * 1e-3) / 1e12, h[1] / (ms * 1e-3) / 1e12, (h[0] + h[1]) / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {2, 4}) {
    run<0>(sms, bps, 0, 4096);
    run<1>(sms, bps, 4096, 0);
    run<2>(sms, bps, 4096, 4096);
    run<2>(sms, bps, 2048, 4096);
  }
  return 0;
}
