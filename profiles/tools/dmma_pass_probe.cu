// Dense-block FP64 tensor-core (DMMA) pass vs the engine's structured pass.
//
// The north star allows "a dense 2^m unitary applied as a batched FP64
// tensor-core contraction, kept only where ncu shows it beats the bandwidth
// kernel". sm_100a's only FP64 MMA is mma.sync.m8n8k4.f64 (tcgen05 has no f64
// kind). This probe runs one pass over a c2-sized state (2^26 complex128,
// 1 GiB) with the engine's tile shape (12 tile bits, one 64 KB tile in
// shared memory per CTA, one CTA per SM) where every phase applies a dense
// 16x16 complex unitary on 4 tile bits as a real 32x32 x 32xN GEMM on DMMA:
//   [Yr; Yi] = [[Ur, -Ui], [Ui, Ur]] [Xr; Xi]
// A fragments (the unitary) stay in registers, B fragments are read from the
// shared-memory tile, D fragments written back in place (each warp owns its
// columns). Phase p uses tile bits 4(p%3)..4(p%3)+3, columns are the other 8.
// Modes: P = 0 (load + store only) and P = 1..6 dense phases; the per-phase
// cost is the slope. Compare with the engine's c2 passes (4-6 phases of
// structured gates, 0.56-0.91 ms per pass, BENCH lines).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_pass_probe dmma_pass_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));       \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

constexpr int T = 12, TILE = 1 << T, THREADS = 512, WARPS = THREADS / 32;

__constant__ double c_ur[32 * 32];  // real form of the 2^M x 2^M complex unitary (row stride 2^(M+1))

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// tile slot of complex row r (M bits at M*q..) and column c (the other bits)
template <int M>
__device__ __forceinline__ unsigned slot_of(unsigned r, unsigned c, int q) {
  const unsigned lo = c & ((1u << (M * q)) - 1);
  return ((c >> (M * q)) << (M * q + M)) | (r << (M * q)) | lo;
}

template <int P, int M>
__global__ void __launch_bounds__(THREADS, 1) pass_kernel(double2* __restrict__ psi, long long ntiles) {
  constexpr int RD = 2 << M;               // real rows / cols of the unitary
  constexpr int MT = RD / 8, KT = RD / 4;  // m8n8k4 tiles
  constexpr int COLS = TILE >> M;          // columns of the tile
  constexpr int NT_W = COLS / WARPS / 8;   // n-tiles per warp
  extern __shared__ __align__(16) double2 tile[];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // A fragments: a[m][k] = Ur[8m + lane/4][4k + lane%4]
  double a[MT][KT];
  if (P > 0) {
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int k = 0; k < KT; ++k) a[m][k] = c_ur[(8 * m + (lane >> 2)) * RD + 4 * k + (lane & 3)];
  }
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const double2* src = psi + (t << T);
#pragma unroll
    for (int j = 0; j < TILE / THREADS; ++j) tile[threadIdx.x + j * THREADS] = src[threadIdx.x + j * THREADS];
    __syncthreads();
#pragma unroll 1
    for (int p = 0; p < P; ++p) {
      const int q = p % (T / M);
#pragma unroll
      for (int nt = 0; nt < NT_W; ++nt) {
        const unsigned c = warp * (NT_W * 8) + nt * 8 + (lane >> 2);
        double d[MT][2];
#pragma unroll
        for (int m = 0; m < MT; ++m) d[m][0] = d[m][1] = 0.0;
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          // B[kk][n]: real row R = 4k + lane%4 of column c
          const unsigned R = 4 * k + (lane & 3);
          const double* base = reinterpret_cast<const double*>(&tile[slot_of<M>(R & ((1u << M) - 1), c, q)]);
          const double b = base[R >> M];
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(d[m], a[m][k], b);
        }
        __syncwarp();
        // D[row 8m + lane/4][col 2(lane%4) + {0,1}]: real row, column
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const unsigned R = 8 * m + (lane >> 2);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const unsigned cc = warp * (NT_W * 8) + nt * 8 + 2 * (lane & 3) + h;
            double* dst = reinterpret_cast<double*>(&tile[slot_of<M>(R & ((1u << M) - 1), cc, q)]);
            dst[R >> M] = d[m][h];
          }
        }
        __syncwarp();
      }
      __syncthreads();
    }
    double2* dst = psi + (t << T);
#pragma unroll
    for (int j = 0; j < TILE / THREADS; ++j) dst[threadIdx.x + j * THREADS] = tile[threadIdx.x + j * THREADS];
    __syncthreads();
  }
}

template <int P, int M>
int timed(double2* d, long long ntiles, int sms, float* ms_out) {
  const size_t smem = TILE * sizeof(double2);
  CK(cudaFuncSetAttribute(pass_kernel<P, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  pass_kernel<P, M><<<sms, THREADS, smem>>>(d, ntiles);
  CK(cudaGetLastError());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) pass_kernel<P, M><<<sms, THREADS, smem>>>(d, ntiles);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms / reps;
  return 0;
}

template <int M>
int sweep(double2* d, long long amps, int sms) {
  // a dense complex unitary: H on each of the M qubits times a diagonal phase
  const int D = 1 << M, RD = 2 * D;
  std::vector<double> ur(RD * RD);
  const double h0 = std::pow(2.0, -0.5 * M);
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      const double h = (__builtin_popcount(i & j) & 1 ? -h0 : h0);
      const double re = h * std::cos(0.1 * j), im = h * std::sin(0.1 * j);
      ur[i * RD + j] = re;
      ur[i * RD + j + D] = -im;
      ur[(i + D) * RD + j] = im;
      ur[(i + D) * RD + j + D] = re;
    }
  CK(cudaMemcpyToSymbol(c_ur, ur.data(), ur.size() * sizeof(double)));
  const long long ntiles = amps >> T;
  float t[7];
  if (timed<0, M>(d, ntiles, sms, &t[0]) || timed<1, M>(d, ntiles, sms, &t[1]) || timed<2, M>(d, ntiles, sms, &t[2]) ||
      timed<3, M>(d, ntiles, sms, &t[3]) || timed<4, M>(d, ntiles, sms, &t[4]) || timed<5, M>(d, ntiles, sms, &t[5]) ||
      timed<6, M>(d, ntiles, sms, &t[6]))
    return 1;
  std::printf("{\"state\": \"2^26 complex128\", \"tile_bits\": 12, \"m\": %d, \"sms\": %d, \"ms_by_dense_phases\": [", M, sms);
  for (int p = 0; p <= 6; ++p) std::printf("%s%.4f", p ? ", " : "", t[p]);
  const double per_phase = (t[6] - t[2]) / 4.0;
  const double flops_phase = double(amps) * 4.0 * RD;  // real RDxRD GEMM per 2^M amplitudes
  std::printf("], \"ms_per_dense_phase\": %.4f, \"dmma_tflops_in_phase\": %.2f, \"hbm_gbs_p0\": %.1f}\n", per_phase,
              flops_phase / (per_phase * 1e-3) / 1e12, 2.0 * amps * 16 / (t[0] * 1e-3) / 1e9);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long amps = 1ll << 26;
  double2* d = nullptr;
  CK(cudaMalloc(&d, amps * sizeof(double2)));
  CK(cudaMemset(d, 0, amps * sizeof(double2)));
  if (sweep<4>(d, amps, sms) || sweep<3>(d, amps, sms)) return 1;
  cudaFree(d);
  return 0;
}
