/*
 * sv_oracle.c -- CPU restatement of the reference hot path in plain C.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline / --impl reference) as the checker or the timed CPU
 * baseline; never linked into libhisvsim.so and never on the product path.
 *
 * Restates, per fixing of the free qubits, the reference's gather ->
 * gates -> scatter (hisim.hier.run_part, pkg/src/hisim/hier.py:220-244;
 * single-fixing form gather/scatter hier.py:112-154) with the per-gate
 * kernels of hisim.statevec (pkg/src/hisim/statevec.py:172-261):
 *   - a 2x2 u on target t (controls must all be 1): pairs at stride 2^t;
 *     if u is diagonal only the non-unit diagonal entries are applied
 *     (statevec.py:177-182), else lo' = u00 lo + u01 hi, hi' = u10 lo + u11 hi;
 *   - SWAP exchanges the 01 and 10 amplitudes (statevec.py:228-238).
 * Gate 2x2s restate statevec.py:31-98. Fixings are independent
 * (SPEC.md:418), so they are spread over POSIX threads (the toolchain here
 * ships no libgomp).
 *
 * Pinned against the reference's golden vectors by tests/test_oracle.py.
 * Build: oracle/Makefile -> oracle/_build/libsv_oracle.so
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>
#include <string.h>
#include <unistd.h>

typedef double complex cplx;

/* same layout as hs_gate in include/hisvsim.h (kind order = GateKind) */
typedef struct {
  int32_t kind, num_slots, slots[3], reserved;
  double params[3];
} or_gate;

enum { H, X, Y, Z, S, T, SDG, TDG, RX, RY, RZ, U1, U3, CX, CZ, CRZ, CRY, SWAP, CCX };

static int controls_of(int kind) {
  return (kind == CX || kind == CZ || kind == CRZ || kind == CRY) ? 1 : kind == CCX ? 2 : 0;
}

/* 2x2 on the target, row-major u[0..3] = u00 u01 u10 u11 */
static void matrix_of(int kind, const double* p, cplx u[4]) {
  const double r = 1.0 / sqrt(2.0);
  double c, s;
  switch (kind) {
    case H: u[0] = r; u[1] = r; u[2] = r; u[3] = -r; return;
    case X: case CX: case CCX: u[0] = 0; u[1] = 1; u[2] = 1; u[3] = 0; return;
    case Y: u[0] = 0; u[1] = -I; u[2] = I; u[3] = 0; return;
    case Z: case CZ: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = -1; return;
    case S: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = I; return;
    case SDG: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = -I; return;
    case T: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = cexp(0.25 * I * M_PI); return;
    case TDG: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = cexp(-0.25 * I * M_PI); return;
    case RX: c = cos(p[0] / 2); s = sin(p[0] / 2);
      u[0] = c; u[1] = -I * s; u[2] = -I * s; u[3] = c; return;
    case RY: case CRY: c = cos(p[0] / 2); s = sin(p[0] / 2);
      u[0] = c; u[1] = -s; u[2] = s; u[3] = c; return;
    case RZ: case CRZ:
      u[0] = cexp(-0.5 * I * p[0]); u[1] = 0; u[2] = 0; u[3] = cexp(0.5 * I * p[0]); return;
    case U1: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = cexp(I * p[0]); return;
    case U3: c = cos(p[0] / 2); s = sin(p[0] / 2);
      u[0] = c; u[1] = -cexp(I * p[2]) * s; u[2] = cexp(I * p[1]) * s; u[3] = cexp(I * (p[1] + p[2])) * c;
      return;
    default: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = 1; return;
  }
}

/* apply one gate to every amplitude pair of a 2^w vector (slots = bits) */
static void apply_gate_block(cplx* v, int w, const or_gate* g) {
  const int64_t dim = (int64_t)1 << w;
  if (g->kind == SWAP) {
    const int64_t a = (int64_t)1 << g->slots[0], b = (int64_t)1 << g->slots[1];
    for (int64_t i = 0; i < dim; ++i)
      if ((i & a) && !(i & b)) {
        const int64_t j = (i ^ a) | b;
        cplx t = v[i]; v[i] = v[j]; v[j] = t;
      }
    return;
  }
  cplx u[4];
  matrix_of(g->kind, g->params, u);
  const int nc = controls_of(g->kind);
  int64_t cmask = 0;
  for (int k = 0; k < nc; ++k) cmask |= (int64_t)1 << g->slots[k];
  const int64_t tb = (int64_t)1 << g->slots[nc];
  const int diag = (u[1] == 0 && u[2] == 0);
  for (int64_t i = 0; i < dim; ++i) {
    if ((i & tb) || (i & cmask) != cmask) continue;
    const int64_t j = i | tb;
    if (diag) {
      if (u[0] != 1.0) v[i] *= u[0];
      if (u[3] != 1.0) v[j] *= u[3];
    } else {
      cplx lo = v[i], hi = v[j];
      v[i] = u[0] * lo + u[1] * hi;
      v[j] = u[2] * lo + u[3] * hi;
    }
  }
}

/* offset of inner index s over positions pos[0..w-1] */
static inline int64_t deposit(int64_t s, const int32_t* pos, int w) {
  int64_t o = 0;
  for (int j = 0; j < w; ++j) o |= ((s >> j) & 1) << pos[j];
  return o;
}

static int g_threads = 0;

int or_num_threads(void) {
  if (g_threads > 0) return g_threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

void or_set_threads(int t) { g_threads = t; }

typedef struct {
  cplx* psi;
  int m, w, nf;
  const int32_t* staged;
  const int32_t* free_pos;
  const or_gate* gates;
  int ngates;
  int64_t begin, end, per_row;
  int err;
} part_job;

static void* part_worker(void* arg) {
  part_job* J = (part_job*)arg;
  const int64_t dim = (int64_t)1 << J->w;
  cplx* blk = (cplx*)malloc(sizeof(cplx) * (size_t)dim);
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)dim);
  if (!blk || !idx) {
    J->err = 2;
  } else {
    for (int64_t s = 0; s < dim; ++s) idx[s] = deposit(s, J->staged, J->w);
    for (int64_t a = J->begin; a < J->end; ++a) {
      const int64_t row = a / J->per_row, f = a % J->per_row;
      const int64_t base = (row << J->m) | deposit(f, J->free_pos, J->nf);
      for (int64_t s = 0; s < dim; ++s) blk[s] = J->psi[base + idx[s]]; /* gather */
      for (int g = 0; g < J->ngates; ++g) apply_gate_block(blk, J->w, &J->gates[g]);
      for (int64_t s = 0; s < dim; ++s) J->psi[base + idx[s]] = blk[s]; /* scatter */
    }
  }
  free(blk);
  free(idx);
  return NULL;
}

/*
 * One part over fixings [fix_begin, fix_begin + fix_count) of a buffer of
 * `rows` x 2^m amplitudes (interleaved re/im doubles). fix_count < 0 means
 * all fixings. Fixing a: row = a >> (m - w), free bits (ascending) = the rest.
 */
int or_run_part(double* data, int m, int64_t rows, const int32_t* staged, int w, const or_gate* gates,
                int ngates, int64_t fix_begin, int64_t fix_count) {
  if (w < 0 || w > m || m > 40) return 1;
  int32_t free_pos[64];
  int nf = 0;
  for (int q = 0, j = 0; q < m; ++q) {
    if (j < w && staged[j] == q) { ++j; continue; }
    free_pos[nf++] = q;
  }
  const int64_t per_row = (int64_t)1 << nf;
  const int64_t total = rows * per_row;
  if (fix_count < 0) fix_count = total - fix_begin;
  if (fix_begin < 0 || fix_begin + fix_count > total) return 1;
  int nt = or_num_threads();
  if (fix_count < nt) nt = fix_count > 0 ? (int)fix_count : 1;
  if (nt > 256) nt = 256;
  pthread_t th[256];
  part_job jobs[256];
  int64_t chunk = (fix_count + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    part_job* J = &jobs[t];
    J->psi = (cplx*)data; J->m = m; J->w = w; J->nf = nf;
    J->staged = staged; J->free_pos = free_pos; J->gates = gates; J->ngates = ngates;
    J->per_row = per_row; J->err = 0;
    J->begin = fix_begin + t * chunk;
    J->end = J->begin + chunk;
    if (J->end > fix_begin + fix_count) J->end = fix_begin + fix_count;
    if (J->begin > J->end) J->begin = J->end;
  }
  for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, part_worker, &jobs[t]);
  part_worker(&jobs[0]);
  int err = jobs[0].err;
  for (int t = 1; t < nt; ++t) {
    pthread_join(th[t], NULL);
    if (jobs[t].err) err = jobs[t].err;
  }
  return err;
}

/* every gate in program order over the whole vector (statevec.simulate_flat) */
int or_simulate_flat(double* data, int n, const or_gate* gates, int ngates) {
  for (int g = 0; g < ngates; ++g) {
    const or_gate* G = &gates[g];
    int32_t staged[3];
    int ns = G->num_slots;
    for (int k = 0; k < ns; ++k) staged[k] = G->slots[k];
    /* sort the operand positions; re-express the gate in slot coordinates */
    for (int a = 0; a < ns; ++a)
      for (int b = a + 1; b < ns; ++b)
        if (staged[b] < staged[a]) { int32_t t = staged[a]; staged[a] = staged[b]; staged[b] = t; }
    or_gate local = *G;
    for (int k = 0; k < ns; ++k)
      for (int j = 0; j < ns; ++j)
        if (staged[j] == G->slots[k]) local.slots[k] = j;
    int e = or_run_part(data, n, 1, staged, ns, &local, 1, 0, -1);
    if (e) return e;
  }
  return 0;
}
