// Tile-movement A/B for the part-pass memory pattern (verdict r1 item 9):
// does a Blackwell bulk-copy / TMA tile loader move a scattered 12-bit tile
// faster than the engine's 16 B cp.async loader? One out-of-place pass over
// a 30-qubit complex128 state (16 GiB in, 16 GiB out), no gates: every CTA
// (one per SM, 3 x 64 KB stages) loads tile t (the 4096 amplitudes whose
// free bits spell t) and writes it back to the same indices of the output.
//
//   ldgsts : 16 B cp.async per thread (LDGSTS) + mbarrier, 16 B st.global
//   bulk   : one cp.async.bulk per contiguous run of the tile (UBLKCP), a
//            bulk store per run (cp.async.bulk.global.shared::cta)
//   tma    : one cp.async.bulk.tensor box per tile (UTMALDG) and one tensor
//            store (UTMASTG), when the tile's runs + free runs fit 5 dims
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_pattern_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int N = 30, T = 12, STAGES = 3, TILE_BYTES = 16 << T, THREADS = 512;

struct Pattern {
  uint64_t tmask;     // tile positions
  int L0;             // length of the tile run starting at position 0
  int nchunk_bits;    // T - L0
  uint64_t chunk_pos; // tile positions >= L0 (deposit target of the chunk index)
  uint64_t free_pos;  // non-tile positions
};

__device__ __forceinline__ uint64_t deposit(uint64_t v, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t m = mask; m; m &= m - 1) {
    if (v & 1) r |= m & (~m + 1);
    v >>= 1;
  }
  return r;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
               :: "r"(smem_u32(b)), "r"(parity) : "memory");
}

// ---- ldgsts: every thread copies 8 x 16 B per tile
__global__ void __launch_bounds__(THREADS, 1) k_ldgsts(const double2* in, double2* out, Pattern P, long long ntiles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * TILE_BYTES);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], THREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto load = [&](long long i) {
    const long long t = blockIdx.x + i * gridDim.x;
    const uint64_t base = deposit(t, P.free_pos);
    const int s = (int)(i % STAGES);
    const unsigned sb = smem_u32(sm + s * TILE_BYTES);
    for (int k = 0; k < (1 << T) / THREADS; ++k) {
      const unsigned e = threadIdx.x + k * THREADS;
      const uint64_t g = base | (e & ((1u << P.L0) - 1)) | deposit(e >> P.L0, P.chunk_pos);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sb + e * 16), "l"(in + g) : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(smem_u32(&full[s])) : "memory");
  };
  for (long long i = 0; i < STAGES && i < mine; ++i) load(i);
  for (long long i = 0; i < mine; ++i) {
    const int s = (int)(i % STAGES);
    mbar_wait(&full[s], (unsigned)((i / STAGES) & 1));
    const long long t = blockIdx.x + i * gridDim.x;
    const uint64_t base = deposit(t, P.free_pos);
    const double2* tile = reinterpret_cast<const double2*>(sm + s * TILE_BYTES);
    for (int k = 0; k < (1 << T) / THREADS; ++k) {
      const unsigned e = threadIdx.x + k * THREADS;
      const uint64_t g = base | (e & ((1u << P.L0) - 1)) | deposit(e >> P.L0, P.chunk_pos);
      out[g] = tile[e];
    }
    __syncthreads();
    if (i + STAGES < mine) load(i + STAGES);
  }
}

// ---- bulk: one bulk copy per contiguous run of 2^L0 amplitudes
__global__ void __launch_bounds__(THREADS, 1) k_bulk(const double2* in, double2* out, Pattern P, long long ntiles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * TILE_BYTES);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int nchunks = 1 << P.nchunk_bits;
  const unsigned run_bytes = 16u << P.L0;
  auto load = [&](long long i) {
    const long long t = blockIdx.x + i * gridDim.x;
    const uint64_t base = deposit(t, P.free_pos);
    const int s = (int)(i % STAGES);
    const unsigned sb = smem_u32(sm + s * TILE_BYTES), bar = smem_u32(&full[s]);
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(TILE_BYTES) : "memory");
    for (int c = threadIdx.x; c < nchunks; c += THREADS) {
      const uint64_t g = base | deposit(c, P.chunk_pos);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(sb + c * run_bytes), "l"(in + g), "r"(run_bytes), "r"(bar) : "memory");
    }
  };
  for (long long i = 0; i < STAGES && i < mine; ++i) load(i);
  for (long long i = 0; i < mine; ++i) {
    const int s = (int)(i % STAGES);
    mbar_wait(&full[s], (unsigned)((i / STAGES) & 1));
    const long long t = blockIdx.x + i * gridDim.x;
    const uint64_t base = deposit(t, P.free_pos);
    const unsigned sb = smem_u32(sm + s * TILE_BYTES);
    for (int c = threadIdx.x; c < nchunks; c += THREADS) {
      const uint64_t g = base | deposit(c, P.chunk_pos);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(out + g), "r"(sb + c * run_bytes), "r"(run_bytes) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
    if (i + STAGES < mine) load(i + STAGES);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- tma: one tensor box per tile (dims: runs of positions, tile runs full, free runs 1)
struct TmaArgs {
  int ndim;
  int free_dim[5];     // which dims are free runs
  int free_shift[5];   // their first free-bit index within t
  int free_len[5];
};

__global__ void __launch_bounds__(THREADS, 1) k_tma(const __grid_constant__ CUtensorMap min, const __grid_constant__ CUtensorMap mout,
                                                   TmaArgs A, long long ntiles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * TILE_BYTES);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&min) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mout) : "memory");
  }
  __syncthreads();
  const long long mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto coords = [&](long long t, int c[5]) {
    for (int d = 0; d < 5; ++d) c[d] = 0;
    for (int f = 0; f < 5; ++f)
      if (A.free_len[f] > 0) c[A.free_dim[f]] = (int)((t >> A.free_shift[f]) & ((1ll << A.free_len[f]) - 1));
  };
  auto load = [&](long long i) {
    const long long t = blockIdx.x + i * gridDim.x;
    int c[5];
    coords(t, c);
    const int s = (int)(i % STAGES);
    const unsigned sb = smem_u32(sm + s * TILE_BYTES), bar = smem_u32(&full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(TILE_BYTES) : "memory");
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 :: "r"(sb), "l"(&min), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar) : "memory");
  };
  if (threadIdx.x == 0)
    for (long long i = 0; i < STAGES && i < mine; ++i) load(i);
  for (long long i = 0; i < mine; ++i) {
    const int s = (int)(i % STAGES);
    if (threadIdx.x == 0) {
      mbar_wait(&full[s], (unsigned)((i / STAGES) & 1));
      const long long t = blockIdx.x + i * gridDim.x;
      int c[5];
      coords(t, c);
      asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                   :: "l"(&mout), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(sm + s * TILE_BYTES)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (i + STAGES < mine) load(i + STAGES);
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// dims (in doubles) of the tile: split positions into runs; tile runs longer
// than the box limit (256) are split. Returns false if more than 5 dims.
bool tma_maps(EncodeFn enc, void* in, void* out, uint64_t tmask, CUtensorMap* mi, CUtensorMap* mo, TmaArgs* A) {
  struct D { bool tile; int start, len; };
  std::vector<D> runs;
  for (int p = 0; p < N;) {
    const bool t = tmask >> p & 1;
    int q = p;
    while (q < N && bool(tmask >> q & 1) == t) ++q;
    int s = p;
    while (s < q) {  // box dims <= 256 elements; dim 0 counts doubles (2 per amplitude)
      const int cap = (t ? (runs.empty() ? 7 : 8) : 30);
      const int len = std::min(q - s, cap);
      runs.push_back({t, s, len});
      s += len;
    }
    p = q;
  }
  if (!runs[0].tile || runs.size() > 5) return false;
  cuuint64_t size[5], stride[4];
  cuuint32_t box[5], es[5];
  const int nd = (int)runs.size();
  memset(A, 0, sizeof(*A));
  A->ndim = nd;
  int fshift = 0, nf = 0;
  for (int d = 0; d < nd; ++d) {
    const D& r = runs[d];
    size[d] = (d == 0 ? 2ull : 1ull) << r.len;
    if (d > 0) stride[d - 1] = (16ull << r.start);
    box[d] = r.tile ? (cuuint32_t)size[d] : 1u;
    es[d] = 1;
    if (!r.tile) {
      A->free_dim[nf] = d;
      A->free_shift[nf] = fshift;
      A->free_len[nf] = r.len;
      fshift += r.len;
      ++nf;
    }
  }
  for (int d = nd; d < 5; ++d) {  // pad to 5 dims of size 1 (stride: the whole state)
    size[d] = 1;
    stride[d - 1] = 16ull << N;
    box[d] = 1;
    es[d] = 1;
  }
  CUresult r1 = enc(mi, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, in, size, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, out, size, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) {
    printf("  tensor map encode failed (%d, %d)\n", (int)r1, (int)r2);
    return false;
  }
  return true;
}

Pattern make_pattern(const std::vector<int>& pos) {
  Pattern P{};
  for (int p : pos) P.tmask |= 1ull << p;
  P.L0 = 0;
  while (P.tmask >> P.L0 & 1) ++P.L0;
  P.nchunk_bits = T - P.L0;
  P.chunk_pos = P.tmask & ~((1ull << P.L0) - 1);
  P.free_pos = ((1ull << N) - 1) & ~P.tmask;
  return P;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = 16ull << N;
  double2 *in, *out;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMemset(in, 0, bytes));
  const int smem = STAGES * TILE_BYTES + 64;
  CK(cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));

  struct Case { const char* name; std::vector<int> pos; };
  std::vector<Case> cases = {
      {"contiguous 0..11", {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11}},
      {"0-2 + 12..20", {0, 1, 2, 12, 13, 14, 15, 16, 17, 18, 19, 20}},
      {"0-2 + 20..28", {0, 1, 2, 20, 21, 22, 23, 24, 25, 26, 27, 28}},
      {"0-5 + 20..25", {0, 1, 2, 3, 4, 5, 20, 21, 22, 23, 24, 25}},
      {"0-3 + 13..20", {0, 1, 2, 3, 13, 14, 15, 16, 17, 18, 19, 20}},
      {"c3 launch 1 (128 B runs, high bits)", {0, 1, 2, 12, 13, 15, 16, 18, 20, 22, 23, 28}},
      {"c3 launch 5 (128 B runs)", {0, 1, 2, 5, 12, 13, 14, 18, 19, 25, 26, 27}},
      {"0-2 + even 12..28", {0, 1, 2, 12, 14, 16, 18, 20, 22, 24, 26, 28}},
      {"0-1 + 12..21 (32 B runs)", {0, 1, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21}},
  };
  const long long ntiles = 1ll << (N - T);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("{\n");
  for (size_t ci = 0; ci < cases.size(); ++ci) {
    const Case& c = cases[ci];
    Pattern P = make_pattern(c.pos);
    CUtensorMap mi, mo;
    TmaArgs A;
    const bool tma_ok = tma_maps(enc, in, out, P.tmask, &mi, &mo, &A);
    double gbs[3] = {0, 0, 0};
    for (int v = 0; v < 3; ++v) {
      if (v == 2 && !tma_ok) continue;
      auto launch = [&]() {
        if (v == 0) k_ldgsts<<<sms, THREADS, smem>>>(in, out, P, ntiles);
        else if (v == 1) k_bulk<<<sms, THREADS, smem>>>(in, out, P, ntiles);
        else k_tma<<<sms, THREADS, smem>>>(mi, mo, A, ntiles);
      };
      for (int w = 0; w < 2; ++w) launch();
      CK(cudaGetLastError());
      CK(cudaEventRecord(e0));
      const int reps = 5;
      for (int r = 0; r < reps; ++r) launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      gbs[v] = 2.0 * bytes / (ms / reps * 1e-3) / 1e9;
    }
    // check the last variant copied the state (input is all zero except a probe)
    printf("  \"%s\": {\"ldgsts_gbs\": %.1f, \"bulk_gbs\": %.1f, \"tma_gbs\": %s, \"run_bytes\": %d, \"tma_dims\": %d}%s\n",
           c.name, gbs[0], gbs[1], tma_ok ? std::to_string(gbs[2]).c_str() : "null", 16 << P.L0, tma_ok ? A.ndim : 0,
           ci + 1 < cases.size() ? "," : "");
  }
  printf("}\n");
  // correctness of each variant on a random-ish input for one pattern
  {
    std::vector<double2> h(1 << 20);
    for (size_t i = 0; i < h.size(); ++i) h[i] = make_double2((double)i, -(double)i);
    CK(cudaMemcpy(in, h.data(), h.size() * 16, cudaMemcpyHostToDevice));
    Pattern P = make_pattern(cases[1].pos);
    CUtensorMap mi, mo;
    TmaArgs A;
    const bool tma_ok = tma_maps(enc, in, out, P.tmask, &mi, &mo, &A);
    for (int v = 0; v < 3; ++v) {
      if (v == 2 && !tma_ok) continue;
      CK(cudaMemset(out, 0xff, 16 << 20));
      if (v == 0) k_ldgsts<<<sms, THREADS, smem>>>(in, out, P, ntiles);
      else if (v == 1) k_bulk<<<sms, THREADS, smem>>>(in, out, P, ntiles);
      else k_tma<<<sms, THREADS, smem>>>(mi, mo, A, ntiles);
      CK(cudaDeviceSynchronize());
      std::vector<double2> g(1 << 20);
      CK(cudaMemcpy(g.data(), out, g.size() * 16, cudaMemcpyDeviceToHost));
      size_t bad = 0;
      for (size_t i = 0; i < g.size(); ++i) bad += g[i].x != h[i].x || g[i].y != h[i].y;
      printf("check variant %d: %zu mismatches in the first 2^20 amplitudes\n", v, bad);
    }
  }
  return 0;
}
