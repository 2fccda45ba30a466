/* A sharded run driven through the C ABI alone (include/hisvsim.h), no
 * Python: 12 qubits over 2 shards of 11 local qubits on one process.
 *
 *   part A   H on qubits 0..10, CX(0,1), RZ(1; 0.7)  (all local; qubit 11 is the rank bit)
 *   switch   qubit 11 (rank bit) <-> qubit 10 (local position 10): hs_group_switch
 *   part B   H(11), CX(11,0), CRZ(11,5; 0.3), U3(3; 0.2,0.4,0.6)  (qubit 11 now at position 10)
 *
 * The shards are compared with a plain host state-vector simulation of the
 * same 12-qubit circuit. Exit code 0 when max |delta| < 1e-12.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include tests/c/group_demo.c \
 *       -L paper_2205_06973_b200/_lib -lhisvsim -L /usr/local/cuda/lib64 -lcudart -lm -o group_demo
 *   ./group_demo [device] [device]      (default: both shards on device 0)
 */
#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "hisvsim.h"

#define N 12
#define NL 11

#define CHECK(call)                                                           \
  do {                                                                        \
    int rc_ = (call);                                                         \
    if (rc_ != HS_OK) {                                                       \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, hs_last_error());  \
      return 2;                                                               \
    }                                                                         \
  } while (0)

typedef double complex cplx;

/* ---- host reference (little-endian: bit q of the index is qubit q) ---- */
static void h1(cplx* s, int q) {
  const double r = 1.0 / sqrt(2.0);
  for (long i = 0; i < (1L << N); ++i)
    if (!(i >> q & 1)) {
      cplx a = s[i], b = s[i | (1L << q)];
      s[i] = r * (a + b);
      s[i | (1L << q)] = r * (a - b);
    }
}
static void u2(cplx* s, int q, const cplx m[4], int ctl) {
  for (long i = 0; i < (1L << N); ++i)
    if (!(i >> q & 1) && (ctl < 0 || (i >> ctl & 1))) {
      cplx a = s[i], b = s[i | (1L << q)];
      s[i] = m[0] * a + m[1] * b;
      s[i | (1L << q)] = m[2] * a + m[3] * b;
    }
}
static void cx(cplx* s, int c, int t) {
  const cplx x[4] = {0, 1, 1, 0};
  u2(s, t, x, c);
}
static void rz(cplx* s, int q, double th, int ctl) {
  const cplx m[4] = {cexp(-I * th / 2), 0, 0, cexp(I * th / 2)};
  u2(s, q, m, ctl);
}
static void u3(cplx* s, int q, double th, double ph, double la) {
  const cplx m[4] = {cos(th / 2), -cexp(I * la) * sin(th / 2), cexp(I * ph) * sin(th / 2),
                     cexp(I * (ph + la)) * cos(th / 2)};
  u2(s, q, m, -1);
}

static hs_gate gate(int kind, int n, int s0, int s1, double p0, double p1, double p2) {
  hs_gate g;
  memset(&g, 0, sizeof(g));
  g.kind = kind;
  g.num_slots = n;
  g.slots[0] = s0;
  g.slots[1] = s1;
  g.params[0] = p0;
  g.params[1] = p1;
  g.params[2] = p2;
  return g;
}

int main(int argc, char** argv) {
  int devs[2] = {argc > 1 ? atoi(argv[1]) : 0, argc > 2 ? atoi(argv[2]) : 0};

  /* part A: staged positions 0..10; slots = positions */
  hs_gate ga[13];
  int ng = 0;
  for (int q = 0; q < NL; ++q) ga[ng++] = gate(HS_H, 1, q, 0, 0, 0, 0);
  ga[ng++] = gate(HS_CX, 2, 0, 1, 0, 0, 0);
  ga[ng++] = gate(HS_RZ, 1, 1, 0, 0.7, 0, 0);
  hs_part pa;
  memset(&pa, 0, sizeof(pa));
  pa.num_staged = NL;
  for (int q = 0; q < NL; ++q) pa.staged[q] = q;
  pa.gate_offset = 0;
  pa.num_gates = ng;

  /* part B after the switch: qubit 11 at position 10; staged {0, 3, 5, 10}
   * -> slots 0: q0, 1: q3, 2: q5, 3: q11 */
  hs_gate gb[4] = {gate(HS_H, 1, 3, 0, 0, 0, 0), gate(HS_CX, 2, 3, 0, 0, 0, 0),
                   gate(HS_CRZ, 2, 3, 2, 0.3, 0, 0), gate(HS_U3, 1, 1, 0, 0.2, 0.4, 0.6)};
  hs_part pb;
  memset(&pb, 0, sizeof(pb));
  pb.num_staged = 4;
  pb.staged[0] = 0;
  pb.staged[1] = 3;
  pb.staged[2] = 5;
  pb.staged[3] = 10;
  pb.num_gates = 4;

  hs_engine* eng[2] = {NULL, NULL};
  hs_program *progA[2], *progB[2];
  for (int r = 0; r < 2; ++r) {
    if (r == 1 && devs[1] == devs[0]) {
      eng[1] = eng[0];
      progA[1] = progA[0];
      progB[1] = progB[0];
      break;
    }
    CHECK(hs_engine_create(devs[r], &eng[r]));
    CHECK(hs_program_create(eng[r], NL, HS_C128, &pa, 1, ga, ng, &progA[r]));
    CHECK(hs_program_create(eng[r], NL, HS_C128, &pb, 1, gb, 4, &progB[r]));
  }
  void* shard[2];
  for (int r = 0; r < 2; ++r) {
    if (cudaSetDevice(devs[r]) != cudaSuccess || cudaMalloc(&shard[r], (size_t)16 << NL) != cudaSuccess) return 3;
  }
  /* |0...0>: amplitude 1 at offset 0 of shard 0 */
  cudaSetDevice(devs[0]);
  CHECK(hs_state_init_basis(shard[0], 1L << NL, HS_C128, 0, NULL));
  cudaSetDevice(devs[1]);
  cudaMemset(shard[1], 0, (size_t)16 << NL);

  void* streams[2] = {NULL, NULL};  /* legacy default streams */
  for (int r = 0; r < 2; ++r) {
    cudaSetDevice(devs[r]);
    CHECK(hs_program_run(progA[r], shard[r], 1, 0, hs_program_num_launches(progA[r]), NULL));
  }
  hs_group* g = NULL;
  CHECK(hs_group_create(2, devs, 4096, &g));
  /* segment bit = position 10; shard r's segment k goes to shard k and lands
   * in the positions of segment r (its old rank-bit value) */
  const int32_t seg_pos[1] = {10};
  const int32_t seg_dst[4] = {0, 1, 0, 1};
  const int32_t src_slot[2] = {0, 1};
  double secs = 0;
  CHECK(hs_group_switch(g, shard, NL, HS_C128, seg_pos, 1, seg_dst, src_slot, streams, &secs));
  for (int r = 0; r < 2; ++r) {
    cudaSetDevice(devs[r]);
    CHECK(hs_program_run(progB[r], shard[r], 1, 0, hs_program_num_launches(progB[r]), NULL));
  }

  cplx* host = calloc(1L << N, sizeof(cplx));
  cplx* got = calloc(1L << NL, sizeof(cplx));
  host[0] = 1;
  for (int q = 0; q < NL; ++q) h1(host, q);
  cx(host, 0, 1);
  rz(host, 1, 0.7, -1);
  h1(host, 11);
  cx(host, 11, 0);
  rz(host, 5, 0.3, 11);
  u3(host, 3, 0.2, 0.4, 0.6);

  double worst = 0;
  for (int r = 0; r < 2; ++r) {
    cudaSetDevice(devs[r]);
    if (cudaMemcpy(got, shard[r], (size_t)16 << NL, cudaMemcpyDeviceToHost) != cudaSuccess) return 3;
    /* shard r: qubit 10 = r (rank bit); positions 0..9 = qubits 0..9,
     * position 10 = qubit 11 */
    for (long o = 0; o < (1L << NL); ++o) {
      long gidx = (o & 0x3FF) | ((long)r << 10) | ((o >> 10 & 1) << 11);
      double d = cabs(got[o] - host[gidx]);
      if (d > worst) worst = d;
    }
  }
  printf("{\"max_abs_delta\": %.3e, \"switch_seconds\": %.3e}\n", worst, secs);
  hs_group_destroy(g);
  for (int r = 0; r < 2; ++r) {
    cudaSetDevice(devs[r]);
    cudaFree(shard[r]);
  }
  for (int r = 0; r < 2; ++r) {
    if (r == 1 && eng[1] == eng[0]) break;
    hs_program_destroy(progA[r]);
    hs_program_destroy(progB[r]);
    hs_engine_destroy(eng[r]);
  }
  free(host);
  free(got);
  return worst < 1e-12 ? 0 : 1;
}
