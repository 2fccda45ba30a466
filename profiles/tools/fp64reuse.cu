#include <cstdio>
#include <cuda_runtime.h>
// DFMA issue rate when the gate constant is a uniform register (kernel
// parameter, ptxas ULDC -> UR operand) vs a vector register (hoisted
// per-thread value): acc = fma(x, c, acc) over 16 accumulators.
//  MODE 0: c uniform, 2 vector operands (x, acc)
//  MODE 1: c in a vector register, one constant for all 16 (reuse possible)
//  MODE 2: c in vector registers, 4 constants rotating (no reuse)
//  MODE 3: 4 uniform constants rotating
template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(double* out, int iters, double c0, double c1, double c2, double c3) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  const double z = (double)(threadIdx.x >> 10);  // 0, not known to ptxas
  double v0 = c0 + z, v1 = c1 + z, v2 = c2 + z, v3 = c3 + z;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int a = (k + 3) & 15;
      if (MODE == 0) x[k] = fma(x[a], c0, x[k]);
      else if (MODE == 1) x[k] = fma(x[a], v0, x[k]);
      else if (MODE == 2) x[k] = fma(x[a], (k & 3) == 0 ? v0 : (k & 3) == 1 ? v1 : (k & 3) == 2 ? v2 : v3, x[k]);
      else x[k] = fma(x[a], (k & 3) == 0 ? c0 : (k & 3) == 1 ? c1 : (k & 3) == 2 ? c2 : c3, x[k]);
    }
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.6789) out[0] = s;
}
template <int M> double run(int sms, int threads) {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096, blocks = sms;
  probe<M><<<blocks, threads>>>(d, 16, 0.999999, 0.999998, 0.999997, 0.999996);
  cudaEventRecord(e0);
  probe<M><<<blocks, threads>>>(d, iters, 0.999999, 0.999998, 0.999997, 0.999996);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * blocks * threads * (double)iters * 16;
  return fl / (ms * 1e-3) / 1e12;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {256, 512})
    printf("threads/SM %d: uniform c %.1f TF | vector c (one) %.1f TF | vector c (4 rotating) %.1f TF | uniform (4 rotating) %.1f TF\n",
           t, run<0>(sms, t), run<1>(sms, t), run<2>(sms, t), run<3>(sms, t));
  return 0;
}
