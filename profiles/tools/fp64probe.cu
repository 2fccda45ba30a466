#include <cstdio>
#include <cuda_runtime.h>
// FP64 issue rate with 1 vs 3 register operands per instruction
template <int MODE>
__global__ void __launch_bounds__(256) probe(double* out, int iters, double a, double b) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (MODE == 0) x[k] = fma(x[k], a, b);                       // 1 register operand
      else if (MODE == 1) x[k] = fma(x[k], x[(k + 5) & 15], b);     // 2 register operands
      else x[k] = fma(x[(k + 3) & 15], x[(k + 7) & 15], x[k]);      // 3 register operands
    }
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.6789) out[0] = s;
}
template <int M> double run(int sms, int blocks_per_sm) {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096, blocks = sms * blocks_per_sm;
  probe<M><<<blocks, 256>>>(d, 16, 0.999999, 1e-7);
  cudaEventRecord(e0);
  probe<M><<<blocks, 256>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * blocks * 256.0 * iters * 16;
  return fl / (ms * 1e-3) / 1e12;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {2, 8}) {
    printf("blocks/SM %d: 1 reg %.1f TF, 2 regs %.1f TF, 3 regs %.1f TF\n", bps, run<0>(sms, bps), run<1>(sms, bps), run<2>(sms, bps));
  }
  return 0;
}
