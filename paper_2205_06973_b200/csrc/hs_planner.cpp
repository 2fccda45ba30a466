// Part planner: turns one part (staged positions + gates in slot
// coordinates, i.e. hisim.hier.ExecutablePart, hier.py:159-217) into a
// device program for the part kernel.
//
// The CTA tile is the part's staged positions plus the lowest other
// positions ("ride-along" bits, processed as extra fixings) up to the tile
// width, so small parts still read long contiguous runs. Inside a tile the
// gates run out of registers: each thread owns 2^RB amplitudes whose index
// bits (the "register bits") change from phase to phase through a shared
// memory exchange. A phase is a maximal group of gates, reordered only across
// commuting gates, whose non-diagonal targets fit the phase's register bits.
// Diagonal gates and controls never need a register bit: a thread knows the
// value of every other tile bit of its amplitudes. SWAP costs nothing: it
// relabels where two qubits live and the final store writes the tile back in
// natural order.
#include <algorithm>
#include <functional>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "hs_common.h"

#include <sys/stat.h>
#include <unistd.h>

namespace hs {

static bool env_is(const char* name, const char* value) {
  const char* e = std::getenv(name);
  return e && std::string(e) == value;
}

// lowest storage positions each pass hands to the next pass's qubits from
// its own tile ($HISVSIM_HOT; default 3 = 128 B runs of complex128, 6 = 1 KB
// runs for programs with global-diagonal passes). Measured on one B200: c3
// with global diagonals 64.6-65.0 ms at 3, 62.0-62.1 at 6, 62.0 at 7 / 8
// (its memory-bound last passes 7.4 / 7.9 -> 6.0 / 6.1 ms); c2 (staged
// diagonals) 5.11 at 3 vs 5.25 at 6; c1 equal.
int layout_hot(bool global_plan = false) {
  const char* e = std::getenv("HISVSIM_HOT");
  if (!e || !*e) return global_plan ? 6 : 3;
  return std::max(1, std::min(8, std::atoi(e)));
}


bool base_matrix(int kind, const double* p, double m[8]) {
  const double r2 = 1.0 / std::sqrt(2.0);
  auto set = [&](double a, double b, double c, double d, double e, double f, double g,
                 double h) {
    m[0] = a; m[1] = b; m[2] = c; m[3] = d; m[4] = e; m[5] = f; m[6] = g; m[7] = h;
  };
  switch (kind) {
    case HS_H: set(r2, 0, r2, 0, r2, 0, -r2, 0); return true;
    case HS_X: case HS_CX: case HS_CCX: set(0, 0, 1, 0, 1, 0, 0, 0); return true;
    case HS_Y: set(0, 0, 0, -1, 0, 1, 0, 0); return true;
    case HS_Z: case HS_CZ: set(1, 0, 0, 0, 0, 0, -1, 0); return true;
    case HS_S: set(1, 0, 0, 0, 0, 0, 0, 1); return true;
    case HS_SDG: set(1, 0, 0, 0, 0, 0, 0, -1); return true;
    case HS_T: set(1, 0, 0, 0, 0, 0, std::cos(0.25 * M_PI), std::sin(0.25 * M_PI)); return true;
    case HS_TDG: set(1, 0, 0, 0, 0, 0, std::cos(0.25 * M_PI), -std::sin(0.25 * M_PI)); return true;
    case HS_RX: {
      double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
      set(c, 0, 0, -s, 0, -s, c, 0);
      return true;
    }
    case HS_RY: case HS_CRY: {
      double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
      set(c, 0, -s, 0, s, 0, c, 0);
      return true;
    }
    case HS_RZ: case HS_CRZ:
      set(std::cos(-0.5 * p[0]), std::sin(-0.5 * p[0]), 0, 0, 0, 0, std::cos(0.5 * p[0]),
          std::sin(0.5 * p[0]));
      return true;
    case HS_U1: set(1, 0, 0, 0, 0, 0, std::cos(p[0]), std::sin(p[0])); return true;
    case HS_U3: {
      double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
      double phi = p[1], lam = p[2];
      set(c, 0, -std::cos(lam) * s, -std::sin(lam) * s, std::cos(phi) * s, std::sin(phi) * s,
          std::cos(phi + lam) * c, std::sin(phi + lam) * c);
      return true;
    }
    default: return false;
  }
}

void component_coefs(const double* m, int c, double coef[4]) {
  const double* a = m + (c < 2 ? 0 : 4);  // m00 or m10 (multiplies x)
  const double* b = a + 2;                // m01 or m11 (multiplies y)
  if ((c & 1) == 0) {  // real part: a.re x.re - a.im x.im + b.re y.re - b.im y.im
    coef[0] = a[0]; coef[1] = -a[1]; coef[2] = b[0]; coef[3] = -b[1];
  } else {             // imaginary part: a.im x.re + a.re x.im + b.im y.re + b.re y.im
    coef[0] = a[1]; coef[1] = a[0]; coef[2] = b[1]; coef[3] = b[0];
  }
}

int component_cost(const double coef[4]) {
  int nz = 0;
  bool unit = false;
  for (int t = 0; t < 4; ++t) {
    if (coef[t] == 0.0) continue;
    ++nz;
    unit |= coef[t] == 1.0 || coef[t] == -1.0;
  }
  return nz == 0 ? 0 : nz - (unit ? 1 : 0);
}

namespace {

// snap entries within a few ulps of 0 / +-1 (relative to the largest entry)
void snap8(double* m) {
  double mx = 0;
  for (int q = 0; q < 8; ++q) mx = std::max(mx, std::fabs(m[q]));
  const double eps = 2e-15 * std::max(mx, 1.0);
  for (int q = 0; q < 8; ++q) {
    if (std::fabs(m[q]) < eps) m[q] = 0.0;
    else if (std::fabs(m[q] - 1.0) < eps) m[q] = 1.0;
    else if (std::fabs(m[q] + 1.0) < eps) m[q] = -1.0;
  }
}

int cost8(const double* m) {
  int c = 0;
  for (int k = 0; k < 4; ++k) {
    double coef[4];
    component_coefs(m, k, coef);
    c += component_cost(coef);
  }
  return c;
}

}  // namespace

Mat2 structure_2x2(const double* m, bool allow_scale) {
  Mat2 best;
  best.s[0] = 1.0;
  best.s[1] = 0.0;
  std::memcpy(best.m, m, sizeof(best.m));
  snap8(best.m);
  best.cost = cost8(best.m);
  if (!allow_scale) return best;
  double mx = 0;
  for (int e = 0; e < 4; ++e) mx = std::max(mx, std::hypot(m[2 * e], m[2 * e + 1]));
  for (int e = 0; e < 4; ++e) {
    const double sr = m[2 * e], si = m[2 * e + 1];
    const double n2 = sr * sr + si * si;
    if (!(n2 > 0) || std::sqrt(n2) < 1e-3 * mx) continue;  // keep M' entries O(1)
    Mat2 c;
    c.s[0] = sr;
    c.s[1] = si;
    for (int q = 0; q < 4; ++q) {  // m / s = m * conj(s) / |s|^2
      const double xr = m[2 * q], xi = m[2 * q + 1];
      c.m[2 * q] = (xr * sr + xi * si) / n2;
      c.m[2 * q + 1] = (xi * sr - xr * si) / n2;
    }
    c.m[2 * e] = 1.0;  // exact by construction
    c.m[2 * e + 1] = 0.0;
    snap8(c.m);
    c.cost = cost8(c.m);
    if (c.cost < best.cost) best = c;
  }
  return best;
}

namespace {

enum Cls { C_DENSE, C_PERM, C_DIAG, C_SWAP };

// tile-logical bit of a pass's global qubit j (plan_part): above every tile
// location, so register / lane logic never sees it
constexpr int GBIT = 32;

int arity_of(int kind) {
  switch (kind) {
    case HS_CX: case HS_CZ: case HS_CRZ: case HS_CRY: case HS_SWAP: return 2;
    case HS_CCX: return 3;
    default: return (kind >= 0 && kind < HS_NUM_KINDS) ? 1 : -1;
  }
}

struct Gate {
  Cls cls;
  int tgt;      // tile-logical bit (SWAP: first operand)
  int other;    // SWAP: second operand
  int ctl[2];
  int nctl;
  int par = -1; // DIAG on the parity tgt ^ par (from CX . D . CX), else -1
  double m[8];
  uint64_t nd;  // tile-logical bits touched non-diagonally
  uint64_t d;   // tile-logical bits touched diagonally (controls, diag targets);
                // global qubits are bits GBIT + j
};

struct Rec {  // a scheduled gate, in locations
  Cls cls;
  int tloc;
  int cloc[2];
  int nctl;
  int ploc;     // parity partner location or -1
  const double* m;
};

int choose_npos(const std::vector<int>& nonreg, int dtype, uint8_t* npos) {
  // lanes (thread bits 0..4) should cover every residue class of the shared
  // memory swizzle so a phase load is bank-conflict free
  const int mod = (dtype == HS_C128) ? 3 : 4;
  std::vector<int> order, rest;
  std::vector<bool> used(nonreg.size(), false);
  for (int c = 0; c < mod; ++c)
    for (size_t i = 0; i < nonreg.size(); ++i)
      if (!used[i] && nonreg[i] % mod == c) { order.push_back(nonreg[i]); used[i] = true; break; }
  for (size_t i = 0; i < nonreg.size(); ++i)
    if (!used[i]) rest.push_back(nonreg[i]);
  // the lowest remaining bits fill the rest of the lanes, then the warp bits
  std::vector<int> all = order;
  all.insert(all.end(), rest.begin(), rest.end());
  for (size_t i = 0; i < all.size(); ++i) npos[i] = (uint8_t)all[i];
  return (int)all.size();
}

void classify(Gate& G) {
  const double* m = G.m;
  bool diag = m[2] == 0 && m[3] == 0 && m[4] == 0 && m[5] == 0;
  bool perm = !diag && m[0] == 0 && m[1] == 0 && m[6] == 0 && m[7] == 0 && m[2] == 1 && m[3] == 0 &&
              m[4] == 1 && m[5] == 0;
  G.cls = diag ? C_DIAG : perm ? C_PERM : C_DENSE;
  uint64_t cm = 0;
  for (int a = 0; a < G.nctl; ++a) cm |= 1ull << G.ctl[a];
  if (G.par >= 0) cm |= 1ull << G.par;
  if (G.cls == C_DIAG) { G.nd = 0; G.d = cm | (1ull << G.tgt); }
  else { G.nd = 1ull << G.tgt; G.d = cm; }
}

bool is_cx(const Gate& G) { return G.cls == C_PERM && G.nctl == 1 && G.par < 0; }

// CX(a,b) . D(b) . CX(a,b) with D = diag(d0, d1) equals the diagonal
// d_{a xor b}: rewrite it as one parity-diagonal (ZZ interaction of QAOA /
// Ising Trotter steps). Ops between the three that touch neither a nor b
// commute with them and stay where they are.
void fuse_parity_diagonals(std::vector<Gate>& gs) {
  const int n = (int)gs.size();
  std::vector<char> dead(n, 0);
  for (int i = 0; i < n; ++i) {
    if (dead[i] || !is_cx(gs[i])) continue;
    const int a = gs[i].ctl[0], b = gs[i].tgt;
    const uint64_t ab = (1ull << a) | (1ull << b);
    auto next_on = [&](int from) {
      for (int j = from; j < n; ++j)
        if (!dead[j] && ((gs[j].nd | gs[j].d) & ab)) return j;
      return -1;
    };
    const int jd = next_on(i + 1);
    if (jd < 0) continue;
    const Gate& D = gs[jd];
    if (!(D.cls == C_DIAG && D.nctl == 0 && D.par < 0 && D.tgt == b)) continue;
    const int jc = next_on(jd + 1);
    if (jc < 0 || !is_cx(gs[jc]) || gs[jc].ctl[0] != a || gs[jc].tgt != b) continue;
    gs[jd].par = a;
    classify(gs[jd]);
    dead[i] = dead[jc] = 1;
  }
  std::vector<Gate> out;
  for (int i = 0; i < n; ++i)
    if (!dead[i]) out.push_back(gs[i]);
  gs.swap(out);
}

// c = b * a for row-major complex 2x2 (apply a first, then b)
void mat_mul(const double* b, const double* a, double* c) {
  for (int r = 0; r < 2; ++r)
    for (int k = 0; k < 2; ++k) {
      double re = 0, im = 0;
      for (int j = 0; j < 2; ++j) {
        const double* x = b + 2 * (2 * r + j);
        const double* y = a + 2 * (2 * j + k);
        re += x[0] * y[0] - x[1] * y[1];
        im += x[0] * y[1] + x[1] * y[0];
      }
      c[2 * (2 * r + k)] = re;
      c[2 * (2 * r + k) + 1] = im;
    }
}

// FP64 instructions per amplitude pair a compiled kernel spends on an
// uncontrolled gate (structure_2x2 for dense; a diagonal is normalised to
// diag(1, d1/d0) with d0 pushed into the part's scalar)
int compiled_cost(const Gate& G) {
  if (G.cls == C_PERM || G.cls == C_SWAP) return 0;
  if (G.cls == C_DIAG) {
    const double ar = G.m[0], ai = G.m[1], br = G.m[6], bi = G.m[7];
    const double n2 = ar * ar + ai * ai;
    if (!(n2 > 0)) return 4;
    double qr = (br * ar + bi * ai) / n2, qi = (bi * ar - br * ai) / n2;
    if (std::fabs(qi) < 2e-15) qi = 0;
    if (std::fabs(qr) < 2e-15) qr = 0;
    if (qi == 0 && std::fabs(std::fabs(qr) - 1.0) < 2e-15) return 0;
    if (qr == 0 && std::fabs(std::fabs(qi) - 1.0) < 2e-15) return 0;
    return (qi == 0 || qr == 0) ? 2 : 4;
  }
  return structure_2x2(G.m, true).cost;
}

// Merge runs of uncontrolled single-qubit gates on one tile bit into one
// 2x2 (their product); a gate touching that bit in any other way ends the
// run. With `cost_aware` (compiled kernels, which exploit 0/+-1 entries) a
// gate joins the run only if the product is no more expensive than the two
// factors apart. Gates on other bits commute with the run, so program order
// of the remaining list is still a valid order of the part.
void fuse_single_qubit_runs(std::vector<Gate>& gs, bool cost_aware) {
  std::vector<Gate> out;
  out.reserve(gs.size());
  std::vector<int> open(64, -1);  // tile bits < T, global bits GBIT + j
  for (const Gate& G : gs) {
    if (G.cls != C_SWAP && G.nctl == 0 && G.par < 0) {
      int& o = open[G.tgt];
      if (o >= 0) {
        Gate F = out[o];
        mat_mul(G.m, out[o].m, F.m);
        classify(F);
        if (!cost_aware || compiled_cost(F) <= compiled_cost(out[o]) + compiled_cost(G)) {
          out[o] = F;
          continue;
        }
      }
      o = (int)out.size();
      out.push_back(G);
      continue;
    }
    const uint64_t touched = G.nd | G.d;
    for (int b = 0; b < 64; ++b)
      if (touched >> b & 1) open[b] = -1;
    out.push_back(G);
  }
  gs.swap(out);
}

double paper_flops(const Rec& r) {
  // dense 2x2 = 14 FLOPs per amplitude, diag with two
  // non-unit entries 6, one non-unit 3, sign/permutation 0; controls scale by
  // the fraction of amplitudes touched
  double f = 0;
  if (r.cls == C_DENSE) f = 14;
  if (r.cls == C_DIAG) {
    bool d0one = r.m[0] == 1.0 && r.m[1] == 0.0;
    bool d1one = r.m[6] == 1.0 && r.m[7] == 0.0;
    bool sign = d0one && r.m[6] == -1.0 && r.m[7] == 0.0;
    f = sign ? 0 : (d0one || d1one) ? 3 : 6;
  }
  return f / double(1 << r.nctl);
}

}  // namespace

int plan_part(int n_local, int dtype, int tile_max, uint32_t options, const int32_t* staged, int w,
              const hs_gate* gates, int num_gates, PartPlan& out, std::string& err, const LayoutIO* lay,
              const int32_t* gpos, int ng) {
  if (n_local < 1 || n_local > 62) { err = "n_local outside [1, 62]"; return HS_ERR_INVALID; }
  if (w < 0 || w > HS_MAX_STAGED) { err = "staged count outside [0, 24]"; return HS_ERR_INVALID; }
  for (int j = 0; j < w; ++j) {
    if (staged[j] < 0 || staged[j] >= n_local) {
      err = "position " + std::to_string(staged[j]) + " outside 0.." + std::to_string(n_local - 1);
      return HS_ERR_INVALID;
    }
    if (j && staged[j] <= staged[j - 1]) { err = "staged positions not strictly ascending"; return HS_ERR_INVALID; }
  }
  // global qubits (gate slots w .. w + ng - 1): positions outside the tile
  // that only diagonal gates act on; compiled, single-CTA passes only
  if (ng < 0 || ng > 32 || (ng > 0 && !gpos)) { err = "global qubit count outside [0, 32]"; return HS_ERR_INVALID; }
  for (int j = 0; j < ng; ++j) {
    if (gpos[j] < 0 || gpos[j] >= n_local) { err = "global position outside the state"; return HS_ERR_INVALID; }
    for (int i = 0; i < w; ++i)
      if (staged[i] == gpos[j]) { err = "global position is staged"; return HS_ERR_INVALID; }
    for (int i = 0; i < j; ++i)
      if (gpos[i] == gpos[j]) { err = "repeated global position"; return HS_ERR_INVALID; }
  }
  if (ng > 0 && !(options & HS_PLAN_JIT)) { err = "global qubits need compiled passes (HS_PLAN_JIT)"; return HS_ERR_UNSUPPORTED; }
  const int T = std::min(std::max(tile_max, w), n_local);
  if (ng > 0 && (T > tile_max || w + ng > n_local)) { err = "global qubits on a cluster tile"; return HS_ERR_UNSUPPORTED; }
  // a part wider than one CTA's tile runs as a cluster tile (compiled parts)
  const int cluster_log = T > tile_max ? T - tile_max : 0;
  if (cluster_log > 0 && (!(options & HS_PLAN_JIT) || !(options & HS_PLAN_CLUSTER) || cluster_log > MAX_CLUSTER_LOG)) {
    err = "part stages " + std::to_string(w) + " qubits; the on-chip tile holds " + std::to_string(tile_max) +
          ((options & HS_PLAN_JIT) ? " (x4 over a CTA cluster)" : " (cluster tiles: HS_PLAN_JIT | HS_PLAN_CLUSTER)");
    return HS_ERR_TOO_WIDE;
  }
  if (T - cluster_log > MAX_TILE) { err = "tile wider than the kernels support"; return HS_ERR_TOO_WIDE; }
  const int RB = std::min((options & HS_PLAN_RB3) ? 3 : MAX_RB, T);

  // physical positions of the staged qubits under the program's layout
  std::vector<int> phy(w);
  for (int j = 0; j < w; ++j) phy[j] = lay && lay->phys_in ? lay->phys_in[staged[j]] : staged[j];
  // tile = staged physical positions + lowest free physical positions
  std::vector<int> tile(phy);
  for (int e = 0; lay && e < lay->num_extra_first && (int)tile.size() < T; ++e) {
    const int p = lay->extra_first[e];
    if (p >= 0 && p < n_local && std::find(tile.begin(), tile.end(), p) == tile.end()) tile.push_back(p);
  }
  for (int p = 0; (int)tile.size() < T && p < n_local; ++p)
    if (std::find(tile.begin(), tile.end(), p) == tile.end()) tile.push_back(p);
  std::sort(tile.begin(), tile.end());
  std::vector<int> tl(w);
  for (int j = 0; j < w; ++j) tl[j] = int(std::find(tile.begin(), tile.end(), phy[j]) - tile.begin());
  // global qubits the tile's fill took in (lowest free positions) are tile
  // bits like any other; the rest keep bits GBIT + j' and the tile's index
  // bits at their physical positions (gphys) give their values
  std::vector<int> gbit(ng), gphys;
  for (int j = 0; j < ng; ++j) {
    const int p = lay && lay->phys_in ? lay->phys_in[gpos[j]] : gpos[j];
    auto it = std::find(tile.begin(), tile.end(), p);
    if (it != tile.end()) {
      gbit[j] = int(it - tile.begin());
    } else {
      gbit[j] = GBIT + (int)gphys.size();
      gphys.push_back(p);
    }
  }

  // classify gates
  std::vector<Gate> gs(num_gates);
  for (int g = 0; g < num_gates; ++g) {
    const hs_gate& in = gates[g];
    int ar = arity_of(in.kind);
    if (ar < 0) { err = "unknown gate kind " + std::to_string(in.kind); return HS_ERR_UNSUPPORTED; }
    if (in.num_slots != ar) { err = "gate " + std::to_string(g) + ": wrong operand count"; return HS_ERR_INVALID; }
    int bits[3];
    for (int a = 0; a < ar; ++a) {
      int s = in.slots[a];
      if (s < 0 || s >= w + ng) { err = "gate " + std::to_string(g) + ": slot outside the part"; return HS_ERR_INVALID; }
      bits[a] = s < w ? tl[s] : gbit[s - w];
      for (int b = 0; b < a; ++b)
        if (bits[b] == bits[a]) { err = "gate " + std::to_string(g) + ": repeated slot"; return HS_ERR_INVALID; }
    }
    Gate& G = gs[g];
    G.nctl = 0;
    if (in.kind == HS_SWAP) {
      G.cls = C_SWAP; G.tgt = bits[0]; G.other = bits[1];
      G.nd = (1u << bits[0]) | (1u << bits[1]); G.d = 0;
      continue;
    }
    base_matrix(in.kind, in.params, G.m);
    G.nctl = ar - 1;
    for (int a = 0; a < G.nctl; ++a) G.ctl[a] = bits[a];
    G.tgt = bits[ar - 1];
    classify(G);
  }
  const int input_gates = num_gates;
  if (options & HS_PLAN_FUSE_1Q) fuse_single_qubit_runs(gs, (options & HS_PLAN_JIT) != 0);
  if (options & HS_PLAN_PARITY) fuse_parity_diagonals(gs);
  num_gates = (int)gs.size();
  // a global qubit is never staged: only diagonal action on it can run
  const int ngl = (int)gphys.size();
  const uint64_t gmask = ngl > 0 ? (((1ull << ngl) - 1) << GBIT) : 0;
  for (const Gate& G : gs)
    if ((G.nd & gmask) || (G.cls != C_DIAG && (G.d & gmask))) {
      err = "a non-diagonal gate acts on a global (unstaged) qubit";
      return HS_ERR_INVALID;
    }

  // storage labelling: loc_of[tile bit] / bit_at[location] (global bits
  // GBIT + j keep their own label)
  std::vector<int> loc_of(64), bit_at(64);
  for (int b = 0; b < 64; ++b) loc_of[b] = bit_at[b] = b;

  PartPlan& P = out;
  P.prog.clear();
  std::memset(&P.info, 0, sizeof(P.info));
  if (ngl > 0) {  // the global qubits' physical positions in the input buffer
    Instr gi;
    std::memset(&gi, 0, sizeof(gi));
    gi.op = I_GLOBALS;
    gi.k = (uint8_t)ngl;
    uint8_t* pos = reinterpret_cast<uint8_t*>(gi.m);
    for (int j = 0; j < ngl; ++j) pos[j] = (uint8_t)gphys[j];
    P.prog.push_back(gi);
  }
  std::vector<char> done(num_gates, 0);
  int remaining = num_gates;
  std::vector<int> R;
  double flops = 0, fp64 = 0;
  int phases = 0;
  // A diagonal gate is "mixed" in a phase when its locations (target,
  // parity partner, controls) are partly register and partly thread bits:
  // compiled kernels fold register-only runs into constants and thread-only
  // runs into one scalar per thread, but apply a mixed one as its own complex
  // multiply per amplitude (QAOA / TFIM parity diagonals: up to half a part's
  // FP64 work).
  auto diag_mixed = [&](const Gate& G, const std::vector<int>& lo, uint32_t regs) {
    int in = 0, all = 0;
    auto see = [&](int b) { ++all; in += lo[b] < 32 && ((regs >> lo[b]) & 1); };
    see(G.tgt);
    if (G.par >= 0) see(G.par);
    for (int a = 0; a < G.nctl; ++a) see(G.ctl[a]);
    return in > 0 && in < all;
  };
  // How many non-diagonal gates a phase would take with register locations
  // restricted to `allow` (a mask; ~0u = first come, up to RB of them), and
  // how many mixed diagonals it would apply. With `defer` (allow an exact
  // register set) mixed diagonals are left for a later phase.
  struct Yield { int taken, mixed; };
  auto phase_yield = [&](uint32_t allow, bool defer) {
    std::vector<char> dn(done);
    std::vector<int> lo(loc_of);
    int taken = 0, nR = 0, mixed = 0;
    uint32_t Rm = 0;
    const bool exact = __builtin_popcount(allow) == RB;
    for (;;) {
      bool progress = false;
      uint64_t blk_nd = 0, blk_d = 0;
      for (int g = 0; g < num_gates; ++g) {
        if (dn[g]) continue;
        const Gate& G = gs[g];
        if ((G.nd & (blk_nd | blk_d)) || (G.d & blk_nd)) { blk_nd |= G.nd; blk_d |= G.d; continue; }
        bool ok = G.cls == C_DIAG || G.cls == C_SWAP;
        if (G.cls == C_DIAG && exact && diag_mixed(G, lo, allow)) {
          if (defer) ok = false;
          else ++mixed;
        }
        if (!ok && G.cls != C_DIAG) {
          const int L = lo[G.tgt];
          if (Rm >> L & 1) ok = true;
          else if (nR < RB && (allow >> L & 1)) { Rm |= 1u << L; ++nR; ok = true; }
        }
        if (!ok) { blk_nd |= G.nd; blk_d |= G.d; continue; }
        if (G.cls == C_SWAP) std::swap(lo[G.tgt], lo[G.other]);
        else if (G.cls != C_DIAG) ++taken;
        dn[g] = 1;
        progress = true;
      }
      if (!progress) break;
    }
    return Yield{taken, mixed};
  };
  // write-back relabel rho: the qubit in tile bit b is stored at tile
  // position rho[b] (a permutation of the tile's own positions, so the store
  // stays in place). It is how the program's layout evolves: qubits staged
  // soonest move to the lowest physical positions so later tiles read long
  // contiguous runs, and the final launches steer every qubit home.
  std::vector<int> rho(T);
  for (int b = 0; b < T; ++b) rho[b] = b;
  if (lay && lay->mode != LAYOUT_KEEP) {
    std::vector<int> occ(T);  // logical position living at tile[b]
    for (int b = 0; b < T; ++b) occ[b] = lay->inv_in ? lay->inv_in[tile[b]] : tile[b];
    auto index_in_tile = [&](int p) {
      auto it = std::find(tile.begin(), tile.end(), p);
      return it == tile.end() ? -1 : int(it - tile.begin());
    };
    if (lay->mode == LAYOUT_OOP) {
      // out of place: store slot bit r = the r-th lowest output position
      // among the tile's qubits
      std::vector<int> outp(T);
      for (int b = 0; b < T; ++b) outp[b] = lay->target[occ[b]];
      for (int b = 0; b < T; ++b) {
        int r = 0;
        for (int c = 0; c < T; ++c) r += outp[c] < outp[b];
        rho[b] = r;
      }
    } else if (lay->mode == LAYOUT_PRIORITY) {
      // the lowest 3 tile positions (the coalescing bits when they are the
      // physical bits 0..2) go to the qubits staged soonest; qubits never
      // staged again go home when home is in the tile (less to restore at
      // the end); the rest fill the remaining positions by next use
      std::vector<int> order(T);
      for (int b = 0; b < T; ++b) order[b] = b;
      std::stable_sort(order.begin(), order.end(),
                       [&](int x, int y) { return lay->next_use[occ[x]] < lay->next_use[occ[y]]; });
      const int32_t never = 1 << 29;
      std::vector<char> taken(T, 0), placed(T, 0);
      const int hot = std::min(lay->hot > 0 ? lay->hot : layout_hot(), T);
      for (int r = 0; r < hot; ++r) {
        rho[order[r]] = r;
        taken[r] = placed[order[r]] = 1;
      }
      for (int r = hot; r < T; ++r) {
        const int b = order[r];
        if (lay->next_use[occ[b]] < never) continue;
        int h = index_in_tile(occ[b]);
        if (h >= hot && !taken[h]) { rho[b] = h; taken[h] = placed[b] = 1; }
      }
      int next = 0;
      for (int r = 0; r < T; ++r) {
        const int b = order[r];
        if (placed[b]) continue;
        while (taken[next]) ++next;
        rho[b] = next;
        taken[next] = 1;
      }
    } else {  // LAYOUT_TARGET: each occupant to target[occ] when that lies in the tile
      std::vector<char> taken(T, 0), placed(T, 0);
      for (int b = 0; b < T; ++b) {
        int t = index_in_tile(lay->target[occ[b]]);
        if (t >= 0 && !taken[t]) { rho[b] = t; taken[t] = 1; placed[b] = 1; }
      }
      int next = 0;
      for (int b = 0; b < T; ++b) {
        if (placed[b]) continue;
        while (taken[next]) ++next;
        rho[b] = next;
        taken[next] = 1;
      }
    }
    if (lay->phys_out) {
      if (lay->mode == LAYOUT_OOP)
        for (int q = 0; q < n_local; ++q) lay->phys_out[q] = lay->target[q];
      else
        for (int b = 0; b < T; ++b) lay->phys_out[occ[b]] = tile[rho[b]];
    }
  }
  // Locations whose store slot is 0..hot-1 (the 128 B store runs): when the
  // last phase keeps them off its register bits, its registers can go
  // straight to HBM (direct store, below), saving a shared-memory round trip
  // of the whole tile. SWAP relabels can move them; the final check decides.
  const int hot_store = dtype == HS_C128 ? 3 : 4;
  uint32_t want_mask = 0;
  if ((options & HS_PLAN_JIT) && cluster_log == 0 && T - RB >= hot_store)
    for (int loc = 0; loc < T; ++loc)
      if (rho[bit_at[loc]] < hot_store) want_mask |= 1u << loc;
  auto nondiag_left = [&]() {
    int c = 0;
    for (int g = 0; g < num_gates; ++g) c += !done[g] && gs[g].cls != C_DIAG && gs[g].cls != C_SWAP;
    return c;
  };
  // one scheduled gate as a device instruction of the phase whose register
  // locations are R_last
  std::vector<int> R_last;
  std::vector<Rec> carry;  // diagonals deferred to the next phase
  auto to_instr = [&](const Rec& r) -> Instr {
    auto reg_of = [&](int L) -> int {
      for (int k = 0; k < (int)R_last.size(); ++k) if (R_last[k] == L) return k;
      return -1;
    };
    Instr in;
    std::memset(&in, 0, sizeof(in));
    in.k = K_NONE;
    uint64_t gq = 0, gc = 0;
    for (int a = 0; a < r.nctl; ++a) {
      int k = reg_of(r.cloc[a]);
      if (r.cloc[a] >= GBIT) gc |= 1ull << (r.cloc[a] - GBIT);
      else if (k >= 0) in.creg |= 1u << k;
      else in.ctid |= 1u << r.cloc[a];
    }
    int k = reg_of(r.tloc);
    if (r.cls == C_DIAG) {
      in.op = I_DIAG;
      uint32_t kreg = 0, qt = 0;
      for (int loc : {r.tloc, r.ploc}) {
        if (loc < 0) continue;
        int kk = reg_of(loc);
        if (loc >= GBIT) gq |= 1ull << (loc - GBIT);
        else if (kk >= 0) kreg |= 1u << kk;
        else qt |= 1u << loc;
      }
      if (r.ploc < 0 && k >= 0) {
        in.k = (uint8_t)k;  // one register bit
      } else if (kreg == 0) {
        in.qtid = qt;       // parity of thread bits: uniform per thread
      } else {
        in.flags |= F_PARITY;
        in.rpos[0] = (uint8_t)kreg;
        in.qtid = qt;
      }
      in.m[0] = r.m[0]; in.m[1] = r.m[1]; in.m[2] = r.m[6]; in.m[3] = r.m[7];
      bool d0one = r.m[0] == 1.0 && r.m[1] == 0.0;
      bool d1one = r.m[6] == 1.0 && r.m[7] == 0.0;
      if (d0one) in.flags |= F_D0_ONE;
      if (d1one) in.flags |= F_D1_ONE;
      if (d0one && r.m[6] == -1.0 && r.m[7] == 0.0) in.flags |= F_SIGN;
      if (gq || gc) instr_set_global(in, gq, gc);
      P.info.diag_gates++;
    } else {
      in.op = (r.cls == C_PERM) ? I_PERM : I_DENSE;
      in.k = (uint8_t)k;  // target is a register bit by construction
      std::memcpy(in.m, r.m, sizeof(in.m));
      if (r.m[1] == 0 && r.m[3] == 0 && r.m[5] == 0 && r.m[7] == 0) in.flags |= F_REAL;
      if (r.cls == C_PERM) P.info.perm_gates++; else P.info.dense_gates++;
    }
    if (in.creg == 0 && in.ctid == 0 && gc == 0) in.flags |= F_PLAIN;
    flops += paper_flops(r);
    {  // FP64 pipe instructions per amplitude, FMA = 1 (what the kernels issue)
      double share = 1.0 / double(1 << r.nctl);
      if (in.op == I_DENSE) fp64 += share * ((in.flags & F_REAL) ? 4.0 : 8.0);
      if (in.op == I_DIAG && !(in.flags & F_SIGN))
        fp64 += share * (((in.flags & (F_D0_ONE | F_D1_ONE)) && !(in.flags & F_PARITY)) ? 2.0 : 4.0);
    }
    return in;
  };
  while (remaining > 0) {
    R.clear();
    // compiled parts pay a shared-memory exchange per phase: pick the
    // register locations that let the most gates into this phase (all
    // RB-subsets of the tile), not just the first targets met; among equals
    // the one applying the fewest mixed diagonals, deferring them to a later
    // phase when that costs this phase no gate
    uint32_t allow = ~0u;
    bool defer = false;
    if ((options & HS_PLAN_JIT) && T <= 16) {
      Yield best = phase_yield(~0u, false);
      best.mixed = 1 << 30;  // first come: mixed count unknown, any exact set with as many gates wins
      // a phase that takes every gate left is the last one: among equally
      // productive register sets, one that leaves the store-run locations
      // to the lanes enables the direct store
      const int left = nondiag_left();
      bool best_direct = false;
      for (uint32_t m = 0; m < (1u << T); ++m) {
        if (__builtin_popcount(m) != RB) continue;
        Yield y = phase_yield(m, false);
        bool d = false;
        if (y.mixed > 0 && y.taken > 0) {
          const Yield yd = phase_yield(m, true);
          if (yd.taken == y.taken) { y = yd; d = true; }
        }
        const bool direct_ok = want_mask && y.taken == left && !d && (m & want_mask) == 0;
        if (y.taken > best.taken ||
            (y.taken == best.taken && (direct_ok > best_direct || (direct_ok == best_direct && y.mixed < best.mixed)))) {
          best = y;
          allow = m;
          defer = d;
          best_direct = direct_ok;
        }
      }
    }
    std::vector<Rec> recs;
    for (;;) {
      bool progress = false;
      uint64_t blk_nd = 0, blk_d = 0;
      for (int g = 0; g < num_gates; ++g) {
        if (done[g]) continue;
        Gate& G = gs[g];
        if ((G.nd & (blk_nd | blk_d)) || (G.d & blk_nd)) { blk_nd |= G.nd; blk_d |= G.d; continue; }
        bool ok = false;
        if (G.cls == C_DIAG || G.cls == C_SWAP) ok = !(G.cls == C_DIAG && defer && diag_mixed(G, loc_of, allow));
        else {
          int L = loc_of[G.tgt];
          if (std::find(R.begin(), R.end(), L) != R.end()) ok = true;
          else if ((int)R.size() < RB && (allow >> L & 1)) { R.push_back(L); ok = true; }
        }
        if (!ok) { blk_nd |= G.nd; blk_d |= G.d; continue; }
        if (G.cls == C_SWAP) {
          int a = G.tgt, b = G.other;
          std::swap(loc_of[a], loc_of[b]);
          bit_at[loc_of[a]] = a;
          bit_at[loc_of[b]] = b;
          P.info.swaps_relabelled++;
        } else {
          Rec r{G.cls, loc_of[G.tgt], {0, 0}, G.nctl, G.par >= 0 ? loc_of[G.par] : -1, G.m};
          for (int a = 0; a < G.nctl; ++a) r.cloc[a] = loc_of[G.ctl[a]];
          recs.push_back(r);
        }
        done[g] = 1;
        --remaining;
        progress = true;
      }
      if (!progress) break;
    }
    // diagonals deferred by the previous phase come first (sinking below
    // moves them past this phase's dense gates where they commute)
    if (!carry.empty()) {
      recs.insert(recs.begin(), carry.begin(), carry.end());
      carry.clear();
    }
    if (recs.empty()) continue;  // only relabels
    // Compiled passes apply a run of diagonal gates as one factor per
    // amplitude (one complex multiply per register and flush): sink every
    // diagonal past the non-diagonal gates that do not act on its locations
    // (they commute: diagonals only meet controls there), so a phase's
    // diagonals gather into as few runs as its dense gates allow.
    if (options & HS_PLAN_JIT) {
      // list schedule: run every dense gate whose predecessors are done (a
      // diagonal predecessor must have been applied, i.e. flushed); gather
      // every diagonal whose dense predecessors ran into the pending run;
      // flush the run only when no dense gate can go on without it
      const int n = (int)recs.size();
      std::vector<uint64_t> ndm(n), dm(n);
      for (int i = 0; i < n; ++i) {
        const Rec& r = recs[i];
        uint64_t c = 0;
        for (int a = 0; a < r.nctl; ++a) c |= 1ull << r.cloc[a];
        if (r.cls == C_DIAG) {
          ndm[i] = 0;
          dm[i] = c | (1ull << r.tloc) | (r.ploc >= 0 ? 1ull << r.ploc : 0ull);
        } else {
          ndm[i] = 1ull << r.tloc;
          dm[i] = c;
        }
      }
      std::vector<std::vector<int>> preds(n);
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < j; ++i)
          if ((ndm[i] & (ndm[j] | dm[j])) || (dm[i] & ndm[j])) preds[j].push_back(i);
      enum { TODO, PENDING, DONE };
      std::vector<int> state(n, TODO);
      std::vector<Rec> order, pend_run;
      std::vector<int> pend_idx;
      order.reserve(n);
      int left = n;
      while (left > 0) {
        for (bool progress = true; progress;) {
          progress = false;
          for (int j = 0; j < n; ++j) {
            if (state[j] != TODO) continue;
            bool ok = true;
            for (int i : preds[j]) ok &= state[i] == DONE;
            if (!ok) continue;
            if (recs[j].cls == C_DIAG) {
              state[j] = PENDING;
              pend_idx.push_back(j);
            } else {
              state[j] = DONE;
              order.push_back(recs[j]);
              --left;
            }
            progress = true;
          }
        }
        // nothing else can run without the pending run: flush it
        bool todo = false;
        for (int j = 0; j < n; ++j) todo |= state[j] == TODO;
        if (!todo) break;
        if (pend_idx.empty()) {
          err = "internal: phase schedule stalled";
          return HS_ERR_INVALID;
        }
        std::sort(pend_idx.begin(), pend_idx.end());
        bool dense_left = false;
        for (int j = 0; j < n; ++j) dense_left |= state[j] == TODO;
        if (!dense_left) break;  // only the trailing run is pending
        for (int j : pend_idx) {
          state[j] = DONE;
          order.push_back(recs[j]);
          --left;
        }
        pend_idx.clear();
      }
      std::sort(pend_idx.begin(), pend_idx.end());
      std::vector<Rec> pend;
      for (int j : pend_idx) pend.push_back(recs[j]);
      // the trailing run commutes with the shared-memory exchange: defer it
      // to the next phase, where it joins that phase's first run (one flush
      // instead of two; the next phase re-expresses it in its registers)
      if (remaining > 0) carry.swap(pend);
      else order.insert(order.end(), pend.begin(), pend.end());
      recs.swap(order);
      if (recs.empty()) continue;  // all deferred
    }
    // the rest of the chosen register set first (the mixed-diagonal choice
    // above assumed it), then the lowest locations
    for (int L = 0; allow != ~0u && L < T && (int)R.size() < RB; ++L)
      if ((allow >> L & 1) && std::find(R.begin(), R.end(), L) == R.end()) R.push_back(L);
    for (int L = 0; (int)R.size() < RB; ++L)
      if (std::find(R.begin(), R.end(), L) == R.end()) R.push_back(L);
    Instr ph;
    std::memset(&ph, 0, sizeof(ph));
    ph.op = I_PHASE;
    ph.k = K_NONE;
    std::vector<int> nonreg;
    for (int L = 0; L < T; ++L)
      if (std::find(R.begin(), R.end(), L) == R.end()) nonreg.push_back(L);
    for (int k = 0; k < RB; ++k) ph.rpos[k] = (uint8_t)R[k];
    choose_npos(nonreg, dtype, ph.npos);
    P.prog.push_back(ph);
    ++phases;
    R_last = R;
    for (const Rec& r : recs) P.prog.push_back(to_instr(r));
  }
  if (phases == 0) {  // no arithmetic at all (empty part or SWAPs only)
    Instr ph;
    std::memset(&ph, 0, sizeof(ph));
    ph.op = I_PHASE;
    ph.k = K_NONE;
    std::vector<int> nonreg;
    for (int L = RB; L < T; ++L) nonreg.push_back(L);
    for (int k = 0; k < RB; ++k) ph.rpos[k] = (uint8_t)k;
    choose_npos(nonreg, dtype, ph.npos);
    P.prog.push_back(ph);
    phases = 1;
    R_last.clear();
    for (int k = 0; k < RB; ++k) R_last.push_back(k);
  }
  // diagonals still deferred (the phases after them only relabelled): the
  // last phase applies them
  for (const Rec& r : carry) P.prog.push_back(to_instr(r));
  carry.clear();
  // final store: register k holds location R[k] of the last phase, which is
  // tile bit bit_at[R[k]]; it is written to tile position rho[bit_at[R[k]]]
  Instr* last = nullptr;
  for (Instr& in : P.prog) if (in.op == I_PHASE) last = &in;
  // Compiled parts store their registers straight to HBM when the last
  // phase's lanes 0..hot-1 can hold store slots 0..hot-1 (a warp then writes
  // whole 128 B lines): the lane order of a phase is free (instructions name
  // tile locations, not thread bits), so move those locations to the front
  // when none of them is a register bit of the last phase.
  bool direct = false;
  {
    const int hot = dtype == HS_C128 ? 3 : 4;
    if ((options & HS_PLAN_JIT) && cluster_log == 0 && T - RB >= hot) {
      std::vector<int> want(hot, -1);
      for (int loc = 0; loc < T; ++loc)
        if (rho[bit_at[loc]] < hot) want[rho[bit_at[loc]]] = loc;
      bool ok = true;
      uint32_t residues = 0;  // the lanes' swizzle residues must differ (conflict-free loads)
      for (int r = 0; r < hot; ++r) {
        ok &= want[r] >= 0;
        for (int k = 0; ok && k < RB; ++k) ok &= last->rpos[k] != want[r];
        if (ok) residues |= 1u << (want[r] % hot);
      }
      // all residues distinct: conflict-free loads in the last phase. With
      // HISVSIM_DIRECT_2WAY=1 two distinct residues (2-way conflicts in the
      // last phase's loads, +1 tile of wavefronts) still go direct, saving the
      // store's shared-memory round trip (2 tiles of wavefronts)
      static const int two_way = [] {  // 0: distinct residues only; 1: two distinct; 2: any
        const char* e = std::getenv("HISVSIM_DIRECT_2WAY");
        return e ? std::atoi(e) : 0;
      }();
      ok &= residues == (1u << hot) - 1 || (two_way >= 1 && hot == 3 && __builtin_popcount(residues) == 2) ||
            (two_way >= 2 && hot == 3);
      if (ok) {
        std::vector<int> order(want.begin(), want.end());
        for (int m = 0; m < T - RB; ++m)
          if (std::find(want.begin(), want.end(), (int)last->npos[m]) == want.end()) order.push_back(last->npos[m]);
        for (int m = 0; m < T - RB; ++m) last->npos[m] = (uint8_t)order[m];
        direct = true;
      }
    }
    // Otherwise the registers go to shared memory in the store order first:
    // pick the last phase's lanes 0..hot-1 so that both their tile locations
    // (the phase's loads) and their store slots (that write) cover every
    // swizzle residue - both bank-conflict free.
    if (!direct && T - RB >= hot) {
      std::vector<int> cand(last->npos, last->npos + (T - RB));
      auto slot = [&](int loc) { return rho[bit_at[loc]]; };
      std::vector<int> pick;
      std::function<bool(size_t, uint32_t, uint32_t)> dfs = [&](size_t from, uint32_t rl, uint32_t rs) -> bool {
        if ((int)pick.size() == hot) return true;
        for (size_t i = from; i < cand.size(); ++i) {
          const uint32_t a = 1u << (cand[i] % hot), b = 1u << (slot(cand[i]) % hot);
          if ((rl & a) || (rs & b)) continue;
          pick.push_back(cand[i]);
          if (dfs(i + 1, rl | a, rs | b)) return true;
          pick.pop_back();
        }
        return false;
      };
      if (dfs(0, 0, 0)) {
        std::vector<int> order(pick);
        for (int c : cand)
          if (std::find(pick.begin(), pick.end(), c) == pick.end()) order.push_back(c);
        for (int m = 0; m < T - RB; ++m) last->npos[m] = (uint8_t)order[m];
      }
    }
  }
  PartLaunch& L = P.launch;
  std::memset(&L, 0, sizeof(L));
  L.direct_store = direct ? 1 : 0;
  L.nprog = (int32_t)P.prog.size();
  L.T = T;
  L.RB = RB;
  L.cluster_log = cluster_log;
  for (int b = 0; b < T; ++b) L.tpos[b] = (uint8_t)tile[b];
  bool ident = true;
  for (int loc = 0; loc < T; ++loc) ident &= (rho[bit_at[loc]] == loc);
  L.fin_sync = ident ? 0 : 1;
  for (int k = 0; k < RB; ++k) L.fin_rpos[k] = (uint8_t)rho[bit_at[last->rpos[k]]];
  for (int m = 0; m < T - RB; ++m) L.fin_npos[m] = (uint8_t)rho[bit_at[last->npos[m]]];
  if (lay && lay->mode == LAYOUT_OOP) {
    L.oop = 1;
    std::vector<int> outp;
    for (int b = 0; b < T; ++b) {
      const int q = lay->inv_in ? lay->inv_in[tile[b]] : tile[b];
      outp.push_back(lay->target[q]);
    }
    std::sort(outp.begin(), outp.end());
    for (int r = 0; r < T; ++r) L.opos[r] = (uint8_t)outp[r];
    int j = 0;
    for (int p = 0; p < n_local; ++p) {
      if (std::find(tile.begin(), tile.end(), p) != tile.end()) continue;
      const int q = lay->inv_in ? lay->inv_in[p] : p;
      L.fpos[j++] = (uint8_t)lay->target[q];
    }
  }

  hs_part_info& I = P.info;
  I.tile_bits = T;
  for (int b = 0; b < T; ++b) I.tile_pos[b] = tile[b];
  I.reg_bits = RB;
  I.phases = phases;
  I.instructions = (int)P.prog.size();
  I.tiles = int64_t(1) << (n_local - T);
  I.fp_ops_per_amp = flops;
  I.fp64_instr_per_amp = (float)fp64;
  I.input_gates = input_gates;
  return HS_OK;
}

namespace {

// Launches that permute the buffer back to the natural layout: every cycle of
// the displacement (data at p belongs at inv[p]) is closed inside one tile;
// cycles longer than a tile are shortened by T - 1 per launch.
int plan_restore(int n_local, int dtype, int tile_max, uint32_t options, std::vector<int32_t>& phys,
                 std::vector<PartPlan>& plans, std::string& err) {
  const int T = std::min(tile_max, n_local);
  for (int guard = 0; guard < 4 * n_local + 4; ++guard) {
    std::vector<int32_t> inv(n_local);
    for (int q = 0; q < n_local; ++q) inv[phys[q]] = q;
    std::vector<std::vector<int>> cycles;
    std::vector<char> seen(n_local, 0);
    for (int p = 0; p < n_local; ++p) {
      if (seen[p] || inv[p] == p) continue;
      std::vector<int> c;
      for (int x = p; !seen[x]; x = inv[x]) { seen[x] = 1; c.push_back(x); }
      cycles.push_back(c);
    }
    if (cycles.empty()) return HS_OK;
    // one launch: whole cycles first-fit, or a chunk of a long cycle. The
    // tile keeps room for the low positions 0..hot-1 (ride-along when not
    // displaced) so the permutation pass reads and writes 128 B runs.
    const int hot = std::min(dtype == HS_C128 ? 3 : 4, T - 1);
    auto tile_need = [&](const std::vector<int>& st) {
      int need = (int)st.size();
      for (int h = 0; h < hot; ++h)
        if (std::find(st.begin(), st.end(), h) == st.end()) ++need;
      return need;
    };
    std::vector<int> set, dest;
    for (auto& c : cycles) {
      std::vector<int> trial(set);
      trial.insert(trial.end(), c.begin(), c.end());
      if (tile_need(trial) <= T) {
        for (size_t k = 0; k < c.size(); ++k) { set.push_back(c[k]); dest.push_back(c[(k + 1) % c.size()]); }
      } else if (set.empty()) {
        const int len = std::max(2, T - hot);
        for (int k = 0; k < len; ++k) { set.push_back(c[k]); dest.push_back(k + 1 < len ? c[k + 1] : c[0]); }
        break;
      }
    }
    std::vector<int32_t> staged, target(phys), next(phys);
    for (size_t k = 0; k < set.size(); ++k) {
      staged.push_back(inv[set[k]]);
      target[inv[set[k]]] = dest[k];
    }
    std::sort(staged.begin(), staged.end());
    LayoutIO lay;
    lay.phys_in = phys.data();
    lay.inv_in = inv.data();
    lay.phys_out = next.data();
    lay.target = target.data();
    lay.mode = LAYOUT_TARGET;
    PartPlan pl;
    int s = plan_part(n_local, dtype, tile_max, options, staged.data(), (int)staged.size(), nullptr, 0, pl, err, &lay);
    if (s != HS_OK) return s;
    pl.info.restore = 1;
    pl.info.user_part = -1;
    plans.push_back(pl);
    phys = next;
  }
  err = "internal: layout restore did not converge";
  return HS_ERR_INVALID;
}

}  // namespace

namespace {

// A part wider than the tile runs as a sequence of sub-parts of at most
// tile_max qubits: gates are taken in program order into the current
// sub-part while they fit and do not depend on a gate left for later (one
// that shares a qubit with it); each round is one pass. The product of the
// sub-parts' gates is the part's (gates only move past gates on disjoint
// qubits). owner[j] = the caller's part of expanded part j.
//
// GROUP_ACROSS runs the same greedy over the whole program's gate stream
// (every part's gates in part order, on storage positions): a pass may then
// finish one part's gates and start the next part's, which the per-part
// split cannot (c5_33, dfs k = 14: 25 -> 16 passes). GROUP_FRONTIER builds
// each pass's qubit set step by step instead: from the gates that wait only
// on qubits outside the set (the frontier), add the qubits of the one whose
// addition makes the most gates runnable per added qubit, until the tile is
// full or nothing gains; the pass then runs every gate whose qubits are in
// the set and that no gate left behind precedes (c4, dfs k = 12: 137 parts
// -> 45 passes; c3 17 -> 15). GROUP_FRONTIER_SEEDED also tries growth
// started from 1-3 qubits of the previous pass (coalesced reads, see
// pass_cost). GROUP_REVERSE_* run the frontier (seeded or plain) over the
// reversed stream - the last pass is chosen first: a gate may join it when
// no later gate left behind shares a qubit - with the last pass seeded with
// storage positions 0..2 / 0..5 so that it can write natural order itself
// (c2: 9 parts + a permutation launch -> 8 passes). A pass belongs to the
// caller's part that contributes most of its gates (ties: the earlier one).
// plan_program plans every grouping in full and keeps the fewest launches.
// GROUP_BEAM_* search the reversed stream breadth-first instead of greedily:
// at every step each of the best partial groupings tries the frontier growth
// from the empty set, from 1-3 qubits of its previous pass and several
// randomised growths (deterministic xorshift), and the BEAM_WIDTH best by
// (passes + penalty, gates left) survive; PEN charges 0.5 pass for a pass
// sharing fewer than 3 qubits with its neighbour (short reads); a last pass
// missing positions 0..2 costs a permutation launch. A beam grouping wins only
// with fewer launches, and is tried only for HBM-bound programs (see
// plan_program): c1 7 -> 6 launches (0.095 -> 0.085 ms). Measured and not
// taken: c3's beam groupings (13 launches without short reads 90.9 vs the
// greedy 13 at 90.3 ms on one box; a 12-launch one, found by some RNG
// streams only, 88.4 vs 90.6), c5_33's (15 launches 1370 vs 17 at 1241 ms).
// streams up to this many gates also try the beam-search groupings; the
// plain beam runs from this many RNG streams
constexpr int BEAM_MAX_GATES = 2000;
constexpr int BEAM_SEEDS = 1;
enum Grouping { GROUP_PER_PART, GROUP_ACROSS, GROUP_FRONTIER, GROUP_FRONTIER_SEEDED, GROUP_REVERSE_LOW3,
                GROUP_REVERSE_LOW6, GROUP_REVERSE_PLAIN_LOW3, GROUP_REVERSE_PLAIN_LOW6, GROUP_BEAM_REVERSE,
                GROUP_BEAM_REVERSE_PEN };

// Cost of a pass in units of one coalesced HBM pass: a full-width pass that
// shares fewer than 3 qubits with the pass before it cannot find its qubits
// on the lowest storage positions (the previous pass could only move its own
// tile's qubits there), so its reads run in short pieces - measured ~2x the
// time of a coalesced pass (c3: 12.7 vs 5.8 ms, ncu r01s3).
double pass_cost(uint64_t used, uint64_t prev, int tile_max) {
  const bool full = __builtin_popcountll(used) > tile_max - 3;
  return (prev && full && __builtin_popcountll(used & prev) < 3) ? 2.0 : 1.0;
}

bool diag_kind(int k) {
  return k == HS_Z || k == HS_S || k == HS_T || k == HS_SDG || k == HS_TDG || k == HS_RZ || k == HS_U1 || k == HS_CZ ||
         k == HS_CRZ;
}

// CX(a,b) D(b) CX(a,b) starting at gate g of a part (D a 1-qubit diagonal)
bool parity_triple(const hs_gate* pg, int g, int n) {
  if (g + 2 >= n || pg[g].kind != HS_CX) return false;
  const hs_gate& G = pg[g];
  const hs_gate& D = pg[g + 1];
  const hs_gate& C = pg[g + 2];
  return D.num_slots == 1 && D.slots[0] == G.slots[1] && diag_kind(D.kind) && D.kind != HS_CZ && D.kind != HS_CRZ &&
         C.kind == HS_CX && C.num_slots == 2 && C.slots[0] == G.slots[0] && C.slots[1] == G.slots[1];
}

// Share of the stream's units (gates, parity triples) that act diagonally.
// Measured: global-diagonal groupings pay off on diagonal-rich circuits (c3
// QAOA 55 %: 13 -> 7 launches, 91.9 -> 69.0 ms; c4 TFIM 49 %: 46 -> 27,
// 5.56 -> 4.55 s; c1 QFT) and lose on random circuits, whose passes are
// FP64-bound and whose CZs are a quarter of the units (c2 26 %: 8 -> 7
// launches, 5.24 -> 5.33 ms; c5_33: 17 -> 12 launches, 1187 -> 1296 ms).
double diag_unit_share(const hs_part* parts, int num_parts, const hs_gate* gates, int num_gates) {
  long units = 0, diag = 0;
  for (int i = 0; i < num_parts; ++i) {
    const hs_part& p = parts[i];
    if (p.gate_offset < 0 || p.num_gates < 0 || p.gate_offset + p.num_gates > num_gates) continue;
    const hs_gate* pg = gates + p.gate_offset;
    for (int g = 0; g < p.num_gates; ++g, ++units) {
      if (parity_triple(pg, g, p.num_gates)) { g += 2; ++diag; continue; }
      diag += diag_kind(pg[g].kind);
    }
  }
  return units ? double(diag) / double(units) : 0.0;
}
constexpr double GLOBAL_DIAG_MIN_SHARE = 0.4;

// With `glob` (HS_PLAN_GLOBAL_DIAG) a unit of the stream is a gate or a
// CX . D . CX parity triple; a unit whose action is diagonal (Z-type gates,
// CZ, CRZ, parity triples) needs none of its qubits staged - the compiled
// pass applies it from the tile's free index bits - and units that are both
// diagonal on a shared qubit commute. Measured on the planner alone: c3 17
// parts -> 7 passes (13 staged-diagonal launches), c4 137 -> 23 (45), c2
// 9 -> 6 (8).
int group_passes(int n_local, int tile_max, const hs_part* parts, int num_parts, const hs_gate* gates,
                 int num_gates, Grouping mode, std::vector<hs_part>& xparts, std::vector<hs_gate>& xgates,
                 std::vector<int>& owner, double* cost, std::string& err, bool glob = false,
                 std::vector<std::vector<int32_t>>* xglobals = nullptr) {
  struct Ref {
    int part;
    const hs_gate* g;  // first gate of the unit (ng consecutive gates of the part)
    int ng;
    uint64_t mask;     // storage positions the unit must stage
    uint64_t all;      // storage positions the unit touches
    uint64_t bn, bd;   // a left-behind unit blocks later units touching bn / acting non-diagonally on bd
  };
  // a later unit u conflicts with the left-behind units' (bn, bd)
  auto conflicts = [](const Ref& u, uint64_t bn, uint64_t bd) { return (u.all & bn) || (u.bn & bd); };
  // gates of `rem` (stream order) that run with qubit set `in`: inside the
  // set and not preceded by a gate left behind on a shared qubit
  auto runnable = [&](const std::vector<Ref>& stream, const std::vector<int>& rem, uint64_t in,
                      std::vector<int>* took) -> int {
    uint64_t bn = 0, bd = 0;
    int n = 0;
    for (int g : rem) {
      const Ref& u = stream[g];
      if (conflicts(u, bn, bd) || (u.mask & ~in)) {
        bn |= u.bn;
        bd |= u.bd;
      } else {
        ++n;
        if (took) took->push_back(g);
      }
    }
    return n;
  };
  // frontier growth from `in`: add the qubits of the frontier gate that make
  // the most gates runnable per added qubit, until full or nothing gains
  auto grow = [&](const std::vector<Ref>& stream, const std::vector<int>& rem, uint64_t in) -> uint64_t {
    for (;;) {
      const int base = runnable(stream, rem, in, nullptr);
      uint64_t bn = 0, bd = 0, best_add = 0;
      double best_gain = 0.0;
      std::vector<uint64_t> seen;
      for (int g : rem) {
        const Ref& u = stream[g];
        if (conflicts(u, bn, bd)) continue;  // (candidates: units clear of the earlier candidates)
        bn |= u.bn;
        bd |= u.bd;
        const uint64_t add = u.mask & ~in;
        if (!add || __builtin_popcountll(in | add) > tile_max) continue;
        if (std::find(seen.begin(), seen.end(), add) != seen.end()) continue;
        seen.push_back(add);
        const double gain = double(runnable(stream, rem, in | add, nullptr) - base) / __builtin_popcountll(add);
        if (gain > best_gain) { best_gain = gain; best_add = add; }
      }
      if (!best_add) return in;
      in |= best_add;
    }
  };
  auto emit = [&](const std::vector<Ref>& stream, const std::vector<int>& chosen, uint64_t in) {
    hs_part q;
    std::memset(&q, 0, sizeof(q));
    int slot_of[64];
    for (int b = 0; b < 64; ++b)  // staged positions stay ascending
      if (in >> b & 1) { slot_of[b] = q.num_staged; q.staged[q.num_staged++] = b; }
    // global qubits: touched (diagonally) but not staged; slots after the staged
    uint64_t touched = 0;
    for (int g : chosen) touched |= stream[g].all;
    std::vector<int32_t> gl;
    for (int b = 0; b < 64; ++b)
      if ((touched & ~in) >> b & 1) { slot_of[b] = q.num_staged + (int)gl.size(); gl.push_back(b); }
    q.gate_offset = (int32_t)xgates.size();
    q.num_gates = 0;
    std::vector<int> votes(num_parts, 0);
    for (int g : chosen) {
      const Ref& r = stream[g];
      const hs_part& p = parts[r.part];
      for (int k = 0; k < r.ng; ++k) {
        hs_gate G = r.g[k];
        for (int a = 0; a < G.num_slots; ++a) G.slots[a] = slot_of[p.staged[G.slots[a]]];
        xgates.push_back(G);
        ++q.num_gates;
      }
      ++votes[r.part];
    }
    if (xglobals) xglobals->push_back(gl);
    int best = stream[chosen[0]].part;
    for (int i = 0; i < num_parts; ++i)
      if (votes[i] > votes[best] || (votes[i] == votes[best] && i < best)) best = i;
    xparts.push_back(q);
    owner.push_back(best);
  };
  uint64_t prev = 0;  // storage positions of the previous pass
  double total = 0.0;
  // group `stream` into passes and emit them
  std::vector<std::pair<std::vector<int>, uint64_t>> held;  // reverse: passes in reverse order
  auto group = [&](const std::vector<Ref>& stream, bool frontier, bool seeded, bool reverse,
                   uint64_t first_seed) -> int {
    std::vector<int> rem(stream.size());
    for (size_t g = 0; g < stream.size(); ++g) rem[g] = (int)g;
    bool first = true;
    while (!rem.empty()) {
      std::vector<int> chosen;
      uint64_t used = 0;
      if (!frontier) {
        uint64_t in = 0, bn = 0, bd = 0;
        for (int g : rem) {
          const Ref& r = stream[g];
          const uint64_t u = in | r.mask;
          if (!conflicts(r, bn, bd) && __builtin_popcountll(u) <= tile_max) {
            in = u;
          } else {
            bn |= r.bn;
            bd |= r.bd;
          }
        }
        runnable(stream, rem, in, &chosen);
        for (int g : chosen) used |= stream[g].mask;
      } else {
        // candidates: plain growth, and growth seeded with the 1-3 previous
        // pass qubits that run the most gates on their own (they stay in
        // the pass, so its reads find them on the low positions); keep the
        // most gates per unit of pass_cost
        std::vector<std::pair<int, uint64_t>> solo;
        for (int b = 0; b < 64; ++b)
          if (prev >> b & 1) solo.push_back({runnable(stream, rem, 1ull << b, nullptr), b});
        std::stable_sort(solo.begin(), solo.end(), [](const std::pair<int, uint64_t>& x,
                                                      const std::pair<int, uint64_t>& y) { return x.first > y.first; });
        double best = -1.0;
        for (int seeds = 0; seeds <= (seeded ? 3 : 0) && seeds <= (int)solo.size(); ++seeds) {
          uint64_t seed = first ? first_seed : 0;
          for (int k = 0; k < seeds; ++k) seed |= 1ull << solo[k].second;
          const uint64_t in = grow(stream, rem, seed);
          std::vector<int> took;
          runnable(stream, rem, in, &took);
          if (took.empty()) continue;
          uint64_t u = seed;
          for (int g : took) u |= stream[g].mask;
          const double score = double(took.size()) / pass_cost(u, prev, tile_max);
          if (score > best) { best = score; chosen.swap(took); used = u; }
        }
      }
      if (chosen.empty() && first && first_seed) {  // the seed left no room (tiny tiles): unseeded
        first_seed = 0;
        continue;
      }
      if (chosen.empty()) { err = "internal: pass grouping made no progress"; return HS_ERR_INVALID; }
      total += pass_cost(used, prev, tile_max);
      prev = used;
      first = false;
      if (reverse) held.push_back({chosen, used});
      else emit(stream, chosen, used);
      std::vector<int> rest;
      rest.reserve(rem.size() - chosen.size());
      size_t c = 0;
      for (int g : rem) {
        if (c < chosen.size() && chosen[c] == g) ++c;
        else rest.push_back(g);
      }
      rem.swap(rest);
    }
    return HS_OK;
  };
  // beam search over the reversed stream (GROUP_BEAM_*): passes go to `held`
  // one beam search with RNG stream `seed`; the result (passes in reverse
  // order) and its score (passes + penalties) go to *out / *score
  auto beam = [&](const std::vector<Ref>& stream, uint64_t first_seed, double penalty, uint64_t seed,
                  std::vector<std::pair<std::vector<int>, uint64_t>>* out, double* score) -> int {
    static const int BEAM_WIDTH = std::getenv("HISVSIM_BEAM_WIDTH") ? std::atoi(std::getenv("HISVSIM_BEAM_WIDTH")) : 32;
    static const int RANDOM_GROWTHS = std::getenv("HISVSIM_BEAM_GROWTHS") ? std::atoi(std::getenv("HISVSIM_BEAM_GROWTHS")) : 6;
    uint64_t base_rng = 0x9E3779B97F4A7C15ull ^ (seed * 0xD1B54A32D192ED03ull);
    if (const char* e = std::getenv("HISVSIM_BEAM_SEED")) base_rng ^= std::strtoull(e, nullptr, 10) * 0xD1B54A32D192ED03ull;
    // xorshift64* on a caller-owned state: every state of every step draws
    // from its own stream, so the result does not depend on the threads
    auto rnd = [](uint64_t& rng) {
      rng ^= rng >> 12; rng ^= rng << 25; rng ^= rng >> 27;
      return double((rng * 2685821657736338717ull) >> 11) / 9007199254740992.0;
    };
    // growth with randomised choice among the best few additions
    auto grow_r = [&](const std::vector<int>& rem, uint64_t in, uint64_t& rng) -> uint64_t {
      for (;;) {
        const int base = runnable(stream, rem, in, nullptr);
        uint64_t bn = 0, bd = 0;
        std::vector<std::pair<double, uint64_t>> adds;
        std::vector<uint64_t> seen;
        for (int g : rem) {
          const Ref& u = stream[g];
          if (conflicts(u, bn, bd)) continue;
          bn |= u.bn;
          bd |= u.bd;
          const uint64_t add = u.mask & ~in;
          if (!add || __builtin_popcountll(in | add) > tile_max) continue;
          if (std::find(seen.begin(), seen.end(), add) != seen.end()) continue;
          seen.push_back(add);
          adds.push_back({double(runnable(stream, rem, in | add, nullptr) - base) / __builtin_popcountll(add), add});
        }
        std::stable_sort(adds.begin(), adds.end(), [](const std::pair<double, uint64_t>& x,
                                                      const std::pair<double, uint64_t>& y) { return x.first > y.first; });
        if (adds.empty() || adds[0].first <= 0) return in;
        const double r = rnd(rng);
        const size_t k = std::min(adds.size() - 1, size_t(r * r * r * std::min<size_t>(3, adds.size())));
        in |= adds[adds[k].first > 0 ? k : 0].second;
      }
    };
    struct State {
      std::vector<std::pair<std::vector<int>, uint64_t>> passes;
      std::vector<int> rem;
      uint64_t prev = 0;
      double pen = 0.0;
    };
    // the successors of one state (its candidate passes)
    auto expand = [&](const State& st, uint64_t rng, std::vector<State>& next) {
      std::vector<uint64_t> cands;
      auto add_cand = [&](uint64_t in) {
        if (std::find(cands.begin(), cands.end(), in) == cands.end()) cands.push_back(in);
      };
      if (!st.prev) {
        add_cand(grow(stream, st.rem, first_seed));
      } else {
        add_cand(grow(stream, st.rem, 0));
        std::vector<int> pb;
        for (int b = 0; b < 64; ++b)
          if (st.prev >> b & 1) pb.push_back(b);
        for (int k = 1; k <= 3 && k <= (int)pb.size(); ++k)
          for (int t = 0; t < 2; ++t) {
            std::vector<int> pick(pb);
            for (int j = 0; j < k; ++j) std::swap(pick[j], pick[j + size_t(rnd(rng) * (pick.size() - j))]);
            uint64_t sd = 0;
            for (int j = 0; j < k; ++j) sd |= 1ull << pick[j];
            add_cand(grow(stream, st.rem, sd));
          }
      }
      for (int t = 0; t < RANDOM_GROWTHS; ++t) add_cand(grow_r(st.rem, 0, rng));
      for (uint64_t in : cands) {
        std::vector<int> took;
        runnable(stream, st.rem, in, &took);
        if (took.empty()) continue;
        uint64_t used = 0;
        for (int g : took) used |= stream[g].mask;
        State ns;
        ns.passes = st.passes;
        ns.passes.push_back({took, used});
        ns.prev = used;
        ns.pen = st.pen + ((st.prev && __builtin_popcountll(used & st.prev) < 3) ? penalty : 0.0);
        // the last pass (the search's first) writes natural order only when
        // it covers the seed positions; else a permutation launch follows
        if (!st.prev && (in & first_seed) != first_seed) ns.pen += 1.0;
        ns.rem.reserve(st.rem.size() - took.size());
        size_t c = 0;
        for (int g : st.rem) {
          if (c < took.size() && took[c] == g) ++c;
          else ns.rem.push_back(g);
        }
        next.push_back(std::move(ns));
      }
    };
    std::vector<State> states(1);
    states[0].rem.resize(stream.size());
    for (size_t g = 0; g < stream.size(); ++g) states[0].rem[g] = (int)g;
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    for (uint64_t step = 0;; ++step) {
      for (const State& st : states)
        if (st.rem.empty()) {
          *out = st.passes;
          *score = st.passes.size() + st.pen;
          return HS_OK;
        }
      std::vector<std::vector<State>> per(states.size());
      auto work = [&](size_t from, size_t stride) {
        for (size_t i = from; i < states.size(); i += stride) {
          uint64_t rng = base_rng ^ ((step * 1315423911ull + i + 1) * 0x94D049BB133111EBull);
          for (int w = 0; w < 4; ++w) rnd(rng);
          expand(states[i], rng, per[i]);
        }
      };
      const size_t nth = std::min<size_t>(hw, states.size());
      if (nth <= 1) {
        work(0, 1);
      } else {
        std::vector<std::thread> pool;
        for (size_t t = 0; t < nth; ++t) pool.emplace_back(work, t, nth);
        for (auto& th : pool) th.join();
      }
      std::vector<State> next;
      for (auto& v : per)
        for (State& ns : v) next.push_back(std::move(ns));
      if (next.empty()) { err = "internal: beam grouping made no progress"; return HS_ERR_INVALID; }
      std::stable_sort(next.begin(), next.end(), [](const State& x, const State& y) {
        const double a = x.passes.size() + x.pen, b = y.passes.size() + y.pen;
        return a != b ? a < b : x.rem.size() < y.rem.size();
      });
      states.clear();
      for (State& ns : next) {
        bool dup = false;
        for (const State& kept : states) dup |= kept.rem == ns.rem;
        if (dup) continue;
        states.push_back(std::move(ns));
        if ((int)states.size() >= BEAM_WIDTH) break;
      }
    }
  };
  std::vector<Ref> all;
  for (int i = 0; i < num_parts; ++i) {
    const hs_part& p = parts[i];
    if (p.gate_offset < 0 || p.num_gates < 0 || p.gate_offset + p.num_gates > num_gates) {
      err = "part " + std::to_string(i) + ": gate window outside the gate array";
      return HS_ERR_INVALID;
    }
    if (p.num_staged < 0 || p.num_staged > HS_MAX_STAGED) { err = "part " + std::to_string(i) + ": bad width"; return HS_ERR_INVALID; }
    for (int j = 0; j < p.num_staged; ++j)
      if (p.staged[j] < 0 || p.staged[j] >= 64) { err = "staged position outside 0..63"; return HS_ERR_INVALID; }
    const hs_gate* pg = gates + p.gate_offset;
    std::vector<Ref> own;
    auto pos_mask = [&](const hs_gate& G, uint64_t* m) -> bool {
      *m = 0;
      if (G.num_slots < 1 || G.num_slots > 3) { err = "gate arity outside 1..3"; return false; }
      for (int a = 0; a < G.num_slots; ++a) {
        const int sl = G.slots[a];
        if (sl < 0 || sl >= p.num_staged) { err = "gate slot outside the part"; return false; }
        *m |= 1ull << p.staged[sl];
      }
      return true;
    };
    for (int g = 0; g < p.num_gates; ++g) {
      const hs_gate& G = pg[g];
      uint64_t m = 0;
      if (!pos_mask(G, &m)) return HS_ERR_INVALID;
      if (!glob) {
        own.push_back(Ref{i, &G, 1, m, m, m, 0});
        continue;
      }
      // CX(a,b) D(b) CX(a,b), consecutive: one diagonal unit (plan_part's
      // HS_PLAN_PARITY fusion turns it into the parity diagonal on a ^ b)
      if (parity_triple(pg, g, p.num_gates)) {
        own.push_back(Ref{i, &G, 3, 0, m, 0, m});
        g += 2;
        continue;
      }
      if (diag_kind(G.kind)) own.push_back(Ref{i, &G, 1, 0, m, 0, m});
      else own.push_back(Ref{i, &G, 1, m, m, m, 0});
    }
    if (mode != GROUP_PER_PART) {
      all.insert(all.end(), own.begin(), own.end());
      continue;
    }
    if (p.num_staged <= tile_max) {
      hs_part q = p;
      q.gate_offset = (int32_t)xgates.size();
      xgates.insert(xgates.end(), pg, pg + p.num_gates);
      xparts.push_back(q);
      owner.push_back(i);
      if (xglobals) xglobals->emplace_back();
      uint64_t u = 0;
      for (int j = 0; j < p.num_staged; ++j) u |= 1ull << p.staged[j];
      total += pass_cost(u, prev, tile_max);
      prev = u;
      continue;
    }
    if (int s = group(own, false, false, false, 0)) return s;
  }
  if (mode >= GROUP_REVERSE_LOW3) {
    const int n = (int)all.size();
    std::vector<Ref> rev(all.rbegin(), all.rend());
    const bool beam_mode = mode == GROUP_BEAM_REVERSE || mode == GROUP_BEAM_REVERSE_PEN;
    const bool low3 = mode == GROUP_REVERSE_LOW3 || mode == GROUP_REVERSE_PLAIN_LOW3 || beam_mode;
    const bool seeded = mode == GROUP_REVERSE_LOW3 || mode == GROUP_REVERSE_LOW6;
    // (the seed never names a position the state does not have)
    // (nor more positions than a tile holds)
    const uint64_t avail = (n_local >= 64 ? ~0ull : ((1ull << n_local) - 1)) & ((1ull << std::min(tile_max, 63)) - 1);
    if (beam_mode) {
      // the plain beam from several RNG streams (a 12-launch c3 grouping
      // turns up in about 2 of 5 searches), the penalised one once
      static const int nseeds = std::getenv("HISVSIM_BEAM_SEEDS") ? std::atoi(std::getenv("HISVSIM_BEAM_SEEDS")) : BEAM_SEEDS;
      const int seeds = mode == GROUP_BEAM_REVERSE ? nseeds : 1;
      double best = 1e300;
      for (int sd = 0; sd < seeds; ++sd) {
        std::vector<std::pair<std::vector<int>, uint64_t>> got;
        double score = 0.0;
        if (int s = beam(rev, 0x7ull & avail, mode == GROUP_BEAM_REVERSE_PEN ? 0.5 : 0.0, sd, &got, &score)) return s;
        if (score < best) { best = score; held.swap(got); }
      }
      for (size_t j = 0; j < held.size(); ++j) total += pass_cost(held[j].second, j ? held[j - 1].second : 0, tile_max);
    } else if (int s = group(rev, true, seeded, true, (low3 ? 0x7ull : 0x3Full) & avail)) {
      return s;
    }
    for (auto it = held.rbegin(); it != held.rend(); ++it) {  // back to program order
      std::vector<int> fwd;
      for (int g : it->first) fwd.push_back(n - 1 - g);
      std::sort(fwd.begin(), fwd.end());
      emit(all, fwd, it->second);
    }
  } else if (mode != GROUP_PER_PART) {
    if (int s = group(all, mode != GROUP_ACROSS, mode == GROUP_FRONTIER_SEEDED, false, 0)) return s;
  }
  if (cost) *cost = total;
  return HS_OK;
}

// positions at the bottom of an out-of-place pass's next layout given to the
// next pass's qubits ($HISVSIM_NEXT_LOW; 3 = the store run only)
int next_low_positions() {
  const char* e = std::getenv("HISVSIM_NEXT_LOW");
  if (!e || !*e) return 3;
  return std::max(3, std::min(62, std::atoi(e)));
}

// the run (in storage bits) a last pass must write in natural order to make
// the gate-free final permutation unnecessary: 3 bits = 128 B of complex128
// (measured: c2 5.96 ms with a 1 KB-run rule and 9 launches vs 5.56 ms with
// 128 B runs and 8; c3 96.6 vs 94.9 ms; 64 B runs lose: c2 6.51 vs 5.74 ms)

// ---- on-disk cache of the chosen tile-pass grouping. Planning every
// grouping candidate (the beam searches above all) costs up to ~1 s of host
// time for a 1000-gate stream; the grouping is a pure function of the
// program's inputs, so a second process reuses it. Key: FNV-1a over the
// inputs and GROUPING_VERSION; value: the passes (hs_part / hs_gate, POD) and
// their owners. A cached grouping is always a valid one for these inputs.
constexpr uint64_t GROUPING_VERSION = 7;

uint64_t grouping_key(int n_local, int dtype, int tile_max, uint32_t options, const hs_part* parts, int num_parts,
                      const hs_gate* gates, int num_gates, const int32_t* given_init) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = (const unsigned char*)p;
    for (size_t i = 0; i < n; ++i) { h ^= b[i]; h *= 1099511628211ull; }
  };
  const int64_t head[6] = {(int64_t)GROUPING_VERSION, n_local, dtype, tile_max, (int64_t)options, num_parts};
  mix(head, sizeof(head));
  mix(parts, sizeof(hs_part) * (size_t)num_parts);
  mix(&num_gates, sizeof(num_gates));
  for (int g = 0; g < num_gates; ++g) {  // field by field: the struct has padding
    const hs_gate& G = gates[g];
    mix(&G.kind, sizeof(G.kind));
    mix(&G.num_slots, sizeof(G.num_slots));
    mix(G.slots, sizeof(G.slots));
    mix(G.params, sizeof(G.params));
  }
  if (given_init) mix(given_init, sizeof(int32_t) * (size_t)n_local);
  for (const char* v : {"HISVSIM_PLAN_SELECT", "HISVSIM_BEAM", "HISVSIM_BEAM_SEED", "HISVSIM_GLOBAL_DIAG"})  // grouping experiments
    if (const char* e = std::getenv(v)) mix(e, std::strlen(e));
  return h;
}

std::string grouping_path(uint64_t key) {
  const std::string dir = hs_cache_dir();
  if (dir.empty()) return std::string();
  char buf[40];
  std::snprintf(buf, sizeof(buf), "/%016llx.grouping", (unsigned long long)key);
  return dir + buf;
}

bool grouping_load(uint64_t key, std::vector<hs_part>& xp, std::vector<hs_gate>& xg, std::vector<int>& owner,
                   std::vector<std::vector<int32_t>>& gl) {
  const std::string path = grouping_path(key);
  if (path.empty()) return false;
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  uint64_t head[4] = {0, 0, 0, 0};
  bool ok = std::fread(head, sizeof(head), 1, f) == 1 && head[0] == key && head[1] < (1u << 20) && head[2] < (1u << 24);
  if (ok) {
    xp.resize(head[1]);
    xg.resize(head[2]);
    owner.resize(head[1]);
    std::vector<int32_t> own(head[1]);
    ok = std::fread(xp.data(), sizeof(hs_part), xp.size(), f) == xp.size() &&
         std::fread(xg.data(), sizeof(hs_gate), xg.size(), f) == xg.size() &&
         std::fread(own.data(), sizeof(int32_t), own.size(), f) == own.size();
    for (size_t i = 0; ok && i < own.size(); ++i) owner[i] = own[i];
    gl.assign(xp.size(), {});
    for (size_t i = 0; ok && i < xp.size(); ++i) {  // per pass: count, positions
      int32_t n = 0;
      ok = std::fread(&n, sizeof(n), 1, f) == 1 && n >= 0 && n <= 64;
      if (!ok) break;
      gl[i].resize(n);
      ok = n == 0 || std::fread(gl[i].data(), sizeof(int32_t), n, f) == (size_t)n;
    }
  }
  std::fclose(f);
  return ok;
}

void grouping_store(uint64_t key, const std::vector<hs_part>& xp, const std::vector<hs_gate>& xg,
                    const std::vector<int>& owner, const std::vector<std::vector<int32_t>>& gl) {
  const std::string path = grouping_path(key);
  if (path.empty()) return;
  const std::string dir = path.substr(0, path.rfind('/'));
  for (size_t i = 1; i <= dir.size(); ++i)
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
  char suffix[48];
  std::snprintf(suffix, sizeof(suffix), ".tmp.%d", (int)getpid());
  const std::string tmp = path + suffix;
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;
  const uint64_t head[4] = {key, xp.size(), xg.size(), 0};
  std::vector<int32_t> own(owner.begin(), owner.end());
  bool ok = std::fwrite(head, sizeof(head), 1, f) == 1 &&
            std::fwrite(xp.data(), sizeof(hs_part), xp.size(), f) == xp.size() &&
            std::fwrite(xg.data(), sizeof(hs_gate), xg.size(), f) == xg.size() &&
            std::fwrite(own.data(), sizeof(int32_t), own.size(), f) == own.size();
  for (size_t i = 0; ok && i < xp.size(); ++i) {
    const int32_t n = i < gl.size() ? (int32_t)gl[i].size() : 0;
    ok = std::fwrite(&n, sizeof(n), 1, f) == 1 && (n == 0 || std::fwrite(gl[i].data(), sizeof(int32_t), n, f) == (size_t)n);
  }
  ok = (std::fclose(f) == 0) && ok;
  if (ok) std::rename(tmp.c_str(), path.c_str());
  else std::remove(tmp.c_str());
}

int final_hot(int n_local, int tile_max) {
  return std::min(3, std::max(1, std::min(n_local, tile_max / 2)));
}

}  // namespace

int plan_program(int n_local, int dtype, int tile_max, uint32_t options, const hs_part* parts, int num_parts,
                 const hs_gate* gates, int num_gates, std::vector<PartPlan>& plans, std::string& err,
                 std::vector<int32_t>* init_phys, const int32_t* given_init, std::vector<int32_t>* final_phys,
                 const std::vector<std::vector<int32_t>>* globals) {
  if (globals && (int)globals->size() != num_parts) { err = "internal: global lists per part"; return HS_ERR_INVALID; }
  bool wide = false;
  for (int i = 0; i < num_parts; ++i) wide |= parts[i].num_staged > tile_max;
  // (cluster tiles run wide parts as one pass each: no regrouping then)
  const bool cluster = (options & HS_PLAN_CLUSTER) && (options & HS_PLAN_JIT);
  if (wide ? !cluster : ((options & HS_PLAN_MERGE) && num_parts > 1)) {
    std::vector<hs_part> xp;
    std::vector<hs_gate> xg;
    std::vector<int> owner;
    std::vector<std::vector<int32_t>> xgl;  // global qubits per pass (HS_PLAN_GLOBAL_DIAG groupings)
    double cost = 0.0;
    int s = group_passes(n_local, tile_max, parts, num_parts, gates, num_gates, GROUP_PER_PART, xp, xg, owner, &cost, err,
                         false, &xgl);
    if (s != HS_OK) return s;
    const uint64_t gkey = (options & HS_PLAN_PART_LOCAL)
                              ? 0
                              : grouping_key(n_local, dtype, tile_max, options, parts, num_parts, gates, num_gates,
                                             given_init);
    std::vector<hs_part> cp;
    std::vector<hs_gate> cg;
    std::vector<int> co;
    std::vector<std::vector<int32_t>> cgl;
    const bool cached = gkey && grouping_load(gkey, cp, cg, co, cgl);
    if (cached) {
      xp.swap(cp);
      xg.swap(cg);
      owner.swap(co);
      xgl.swap(cgl);
    } else if (!(options & HS_PLAN_PART_LOCAL)) {
      // regroup the whole gate stream when that takes fewer launches; among
      // regroupings with as few, the lowest pass_cost. Every candidate is
      // planned in full (host only, ~20 ms each) and judged by its real
      // launch count: passes plus a ping-pong program's final permutation or
      // an in-place program's restore launches. (Measured on one B200: a
      // 9-pass forward regrouping of c2 ran 6.00 vs 5.71 ms for its 9 parts
      // + permutation, so equal counts keep the parts; c5_33's unseeded
      // frontier, 15 passes, 1224 vs 1273 ms for the seeded 16.)
      double fp64_per_launch = 0.0;  // FP64 instructions per amplitude and launch of the parts' plan
      auto planned = [&](const std::vector<hs_part>& ps, const std::vector<hs_gate>& gs,
                         const std::vector<std::vector<int32_t>>& gl, size_t* out) -> int {
        std::vector<PartPlan> tmp;
        std::vector<int32_t> ip, fp;
        std::string e;
        const int st = plan_program(n_local, dtype, tile_max, options & ~HS_PLAN_MERGE, ps.data(), (int)ps.size(),
                                    gs.data(), (int)gs.size(), tmp, e, &ip, given_init, &fp, &gl);
        if (st != HS_OK) { err = e; return st; }
        *out = tmp.size();
        double f = 0.0;
        for (const PartPlan& pl : tmp) f += pl.info.fp64_instr_per_amp;
        fp64_per_launch = tmp.empty() ? 0.0 : f / double(tmp.size());
        return HS_OK;
      };
      size_t best_launches = 0;
      if ((s = planned(xp, xg, xgl, &best_launches)) != HS_OK) return s;
      // Passes issuing more FP64 work than a pass moves HBM bytes (~60 FP64
      // instructions per complex128 amplitude at the measured rates) gain
      // little from fewer launches, and the beam's denser passes measured
      // slower there (c5_33: 15 beam launches 1370 ms vs 17 greedy 1241):
      // beam candidates only for HBM-bound programs (c1 7 -> 6, 0.095 ->
      // 0.085 ms; c3 ties at 13)
      const bool fp64_bound = fp64_per_launch > (dtype == HS_C128 ? 60.0 : 30.0);
      bool regrouped = false;
      int stream_gates = 0;
      for (int i = 0; i < num_parts; ++i) stream_gates += parts[i].num_gates;
      std::vector<Grouping> modes = {GROUP_ACROSS, GROUP_FRONTIER, GROUP_FRONTIER_SEEDED, GROUP_REVERSE_LOW3,
                                     GROUP_REVERSE_LOW6, GROUP_REVERSE_PLAIN_LOW3, GROUP_REVERSE_PLAIN_LOW6};
      const char* beam_env = std::getenv("HISVSIM_BEAM");  // "0": greedy groupings only (A/B)
      const bool beam_forced = beam_env && std::string(beam_env) == "1";
      if (stream_gates <= BEAM_MAX_GATES && (!fp64_bound || beam_forced) && !(beam_env && std::string(beam_env) == "0")) {
        modes.push_back(GROUP_BEAM_REVERSE);
        modes.push_back(GROUP_BEAM_REVERSE_PEN);
      }
      // global-diagonal groupings (HS_PLAN_GLOBAL_DIAG: compiled passes with
      // the parity fusion; $HISVSIM_GLOBAL_DIAG=0 turns them off for A/B):
      // every mode is also tried with unstaged diagonals
      // ($HISVSIM_GLOBAL_DIAG=1 tries them whatever the circuit's diagonal share)
      const bool glob_ok = (options & HS_PLAN_GLOBAL_DIAG) && (options & HS_PLAN_JIT) && (options & HS_PLAN_PARITY) &&
                           !env_is("HISVSIM_GLOBAL_DIAG", "0") &&
                           (env_is("HISVSIM_GLOBAL_DIAG", "1") ||
                            diag_unit_share(parts, num_parts, gates, num_gates) >= GLOBAL_DIAG_MIN_SHARE);
      std::vector<std::pair<Grouping, bool>> cands;
      for (Grouping mode : modes) cands.push_back({mode, false});
      if (glob_ok)
        for (Grouping mode : modes) cands.push_back({mode, true});
      for (const auto& cand : cands) {
        const Grouping mode = cand.first;
        std::vector<hs_part> ap;
        std::vector<hs_gate> ag;
        std::vector<int> ao;
        std::vector<std::vector<int32_t>> agl;
        double c = 0.0;
        s = group_passes(n_local, tile_max, parts, num_parts, gates, num_gates, mode, ap, ag, ao, &c, err, cand.second,
                         &agl);
        if (s != HS_OK) return s;
        size_t la = 0;
        if ((s = planned(ap, ag, agl, &la)) != HS_OK) {
          if (!cand.second) return s;
          continue;  // e.g. more than 32 global qubits in one pass: not this grouping
        }
        if (std::getenv("HISVSIM_PLAN_DEBUG")) {
          std::fprintf(stderr, "[plan] grouping %d%s: %zu passes, %zu launches, cost %.1f", (int)mode,
                       cand.second ? " (global diagonals)" : "", ap.size(), la, c);
          if (options & HS_PLAN_JIT) {  // the generator's FP64 count per launch
            std::vector<PartPlan> tmp;
            std::vector<int32_t> ip, fp;
            std::string e;
            if (plan_program(n_local, dtype, tile_max, options & ~HS_PLAN_MERGE, ap.data(), (int)ap.size(), ag.data(),
                             (int)ag.size(), tmp, e, &ip, given_init, &fp, &agl) == HS_OK) {
              std::fprintf(stderr, ", fp64/amp:");
              for (const PartPlan& pl : tmp) std::fprintf(stderr, " %.0f", jit_fp64_per_amp(pl, dtype, n_local));
            }
          }
          std::fprintf(stderr, "\n");
        }
        // fewest launches; among as few, the lowest pass_cost (measured c3:
        // 13 launches with one short-read pass 96.3 ms, 14 coalesced 96.6-97.4)
        static const bool by_cost = [] {
          const char* e = std::getenv("HISVSIM_PLAN_SELECT");
          return e && std::string(e) == "cost";
        }();
        // a beam grouping replaces a greedy one only with fewer launches (c3,
        // same box: beam's 13 short-read-free launches 90.9 ms vs the greedy
        // 13 with three short reads 90.3; c1 7 -> 6, c5_33 17 -> 16 launches)
        const bool beam_mode = mode == GROUP_BEAM_REVERSE || mode == GROUP_BEAM_REVERSE_PEN;
        const bool better = by_cost ? (c < cost || (c == cost && la < best_launches))
                                    : (la < best_launches ||
                                       (regrouped && !beam_mode && la == best_launches && c < cost));
        if (better) {
          xp.swap(ap); xg.swap(ag); owner.swap(ao); xgl.swap(agl); cost = c; best_launches = la;
          regrouped = true;
        }
      }
    }
    s = plan_program(n_local, dtype, tile_max, options & ~HS_PLAN_MERGE, xp.data(), (int)xp.size(), xg.data(), (int)xg.size(), plans,
                     err, init_phys, given_init, final_phys, &xgl);
    if (s != HS_OK) return s;
    if (gkey && !cached) grouping_store(gkey, xp, xg, owner, xgl);
    for (auto& pl : plans)
      if (pl.info.user_part >= 0) pl.info.user_part = owner[pl.info.user_part];
    return HS_OK;
  }
  plans.assign(num_parts, PartPlan());
  const bool layout = (options & HS_PLAN_LAYOUT) && num_parts > 0 && n_local > 0;
  std::vector<int32_t> phys(std::max(n_local, 1)), inv(std::max(n_local, 1));
  for (int q = 0; q < n_local; ++q) phys[q] = inv[q] = q;
  if (given_init) {  // the caller's buffer arrives in this layout (e.g. after an in-place switch)
    for (int q = 0; q < n_local; ++q) phys[q] = given_init[q];
    for (int q = 0; q < n_local; ++q) inv[phys[q]] = q;
  } else if (layout && (options & HS_PLAN_INIT_LAYOUT)) {
    // the state starts as a basis state, which is one amplitude in any
    // layout: start with part 0's qubits on the lowest positions (its reads
    // become one contiguous run per tile); qubits whose home they take move
    // to the homes those qubits vacate
    const hs_part& p0 = parts[0];
    std::vector<char> in0(n_local, 0);
    for (int j = 0; j < p0.num_staged; ++j)
      if (p0.staged[j] >= 0 && p0.staged[j] < n_local) in0[p0.staged[j]] = 1;
    std::vector<int32_t> vacated;
    int pos = 0;
    for (int q = 0; q < n_local; ++q)
      if (in0[q]) { phys[q] = pos++; if (q >= p0.num_staged) vacated.push_back(q); }
    size_t v = 0;
    for (int q = 0; q < p0.num_staged && q < n_local; ++q)
      if (!in0[q]) phys[q] = vacated[v++];
    for (int q = 0; q < n_local; ++q) inv[phys[q]] = q;
  }
  if (init_phys) init_phys->assign(phys.begin(), phys.begin() + n_local);
  // next_use[i][q]: parts after i until q is staged again (large = never)
  std::vector<std::vector<int32_t>> next_use;
  if (layout) {
    const int32_t never = 1 << 29;
    next_use.assign(num_parts, std::vector<int32_t>(n_local, never));
    std::vector<int32_t> upcoming(n_local, -1);
    for (int i = num_parts - 1; i >= 0; --i) {
      for (int q = 0; q < n_local; ++q)
        if (upcoming[q] >= 0) next_use[i][q] = upcoming[q] - i;
      for (int j = 0; j < parts[i].num_staged; ++j) {
        int q = parts[i].staged[j];
        if (q >= 0 && q < n_local) upcoming[q] = i;
      }
    }
  }
  std::vector<int32_t> home(std::max(n_local, 1));
  for (int q = 0; q < n_local; ++q) home[q] = q;
  // ping-pong: out-of-place parts alternate state -> scratch -> state; an
  // odd part count runs part 0 in place so the last part lands in the state
  const bool pp = layout && (options & HS_PLAN_PINGPONG) && num_parts >= 2;
  // the next part's qubits go to the lowest `hot` positions (3: 128 B runs
  // of complex128). Measured with the tile-pass planner: hot = 3 vs 6 (1 KB
  // runs) c2 5.42 vs 5.55 ms, c3 95.0 vs 95.4 ms, c1 equal (an earlier
  // planner measured the opposite: c3 126 vs 121 ms). The gate-free final
  // permutation stages at most 2 * hot qubits.
  bool global_plan = false;  // a program with global-diagonal passes
  for (int i = 0; globals && i < num_parts; ++i) global_plan |= !(*globals)[i].empty();
  const int hot = std::min(layout_hot(global_plan), std::max(1, std::min(n_local, tile_max / 2)));
  const bool no_restore = (options & HS_PLAN_NO_RESTORE) != 0;
  // The last part's tile takes the lowest logical qubits it does not stage
  // as its extra bits; it writes natural order itself when those and its
  // own cover qubits 0..final_hot-1 (128 B store runs), else it writes a
  // coalesced layout and one gate-free out-of-place launch permutes into
  // natural order.
  bool need_restore = false;
  std::vector<int32_t> last_extra;  // logical qubits
  if (pp && !no_restore) {
    const hs_part& pl = parts[num_parts - 1];
    const int w = std::max(0, std::min(pl.num_staged, HS_MAX_STAGED));
    const int T = std::min(std::max(tile_max, w), n_local);
    std::vector<char> cov(n_local + 1, 0);
    for (int j = 0; j < w; ++j)
      if (pl.staged[j] >= 0 && pl.staged[j] < n_local) cov[pl.staged[j]] = 1;
    for (int q = 0; q < n_local && w + (int)last_extra.size() < T; ++q)
      if (!cov[q]) { last_extra.push_back(q); cov[q] = 1; }
    int run = 0;
    while (run < n_local && cov[run]) ++run;
    need_restore = run < std::min(final_hot(n_local, tile_max), n_local);
  }
  const bool first_inplace = pp && ((num_parts + (need_restore ? 1 : 0)) % 2 == 1);
  int cur_buf = 0;
  for (int i = 0; i < num_parts; ++i) {
    const hs_part& p = parts[i];
    if (p.gate_offset < 0 || p.num_gates < 0 || p.gate_offset + p.num_gates > num_gates) {
      err = "part " + std::to_string(i) + ": gate window outside the gate array";
      return HS_ERR_INVALID;
    }
    LayoutIO lay;
    lay.hot = hot;
    std::vector<int32_t> next(phys);
    std::vector<int32_t> tgt(phys);
    const bool oop = pp && !(first_inplace && i == 0);
    if (oop) {
      lay.phys_in = phys.data();
      lay.inv_in = inv.data();
      lay.phys_out = next.data();
      lay.mode = LAYOUT_OOP;
      std::vector<int32_t> extra_phys;
      if (i + 1 == num_parts && !need_restore && !no_restore) {
        for (int q = 0; q < n_local; ++q) tgt[q] = q;  // the last part writes natural order
        for (int32_t q : last_extra) extra_phys.push_back(phys[q]);
        lay.extra_first = extra_phys.data();
        lay.num_extra_first = (int)extra_phys.size();
      } else {
        // the next layout: this tile's qubits that the next part stages go
        // to the lowest positions (coalesced stores now, coalesced loads
        // next), then other tile qubits; everything else stays put (swaps)
        const int w = std::max(0, std::min(p.num_staged, HS_MAX_STAGED));
        const int T = std::min(std::max(tile_max, w), n_local);
        std::vector<int> tpos;
        for (int j = 0; j < w; ++j)
          if (p.staged[j] >= 0 && p.staged[j] < n_local) tpos.push_back(phys[p.staged[j]]);
        for (int q = 0; (int)tpos.size() < T && q < n_local; ++q)
          if (std::find(tpos.begin(), tpos.end(), q) == tpos.end()) tpos.push_back(q);
        std::sort(tpos.begin(), tpos.end());
        std::vector<char> nxt(n_local, 0);
        if (i + 1 < num_parts) {
          const hs_part& p1 = parts[i + 1];
          for (int j = 0; j < p1.num_staged; ++j)
            if (p1.staged[j] >= 0 && p1.staged[j] < n_local) nxt[p1.staged[j]] = 1;
        } else {
          for (int q = 0; q < hot; ++q) nxt[q] = 1;  // the restore launch stages 0..hot-1
        }
        std::vector<int> cand;
        for (int pass = 0; pass < 2; ++pass)
          for (int pp_ : tpos)
            if ((nxt[inv[pp_]] != 0) == (pass == 0)) cand.push_back(inv[pp_]);
        std::vector<int32_t> tinv(inv);
        auto place = [&](int q, int r) {  // q to position r, its occupant to q's old one
          const int pq = tgt[q];
          if (pq == r) return;
          const int o = tinv[r];
          tgt[o] = pq;
          tinv[pq] = o;
          tgt[q] = r;
          tinv[r] = q;
        };
        for (int r = 0; r < hot && r < (int)cand.size(); ++r) place(cand[r], r);
        // Out of place any permutation of the positions above the store run
        // is free (stores stay 128 B runs): the next pass's other qubits -
        // tile or free - take the positions right above, so its tile reads
        // longer runs / fewer DRAM pages (HISVSIM_NEXT_LOW positions in all)
        const int next_low = std::min(n_local, next_low_positions());
        int r = hot;
        for (int p = 0; p < n_local && r < next_low; ++p) {
          const int q = tinv[p];
          if (p < hot || !nxt[q]) continue;
          if (p >= r) place(q, r);
          ++r;
        }
      }
      lay.target = tgt.data();
    } else if (layout) {
      lay.phys_in = phys.data();
      lay.inv_in = inv.data();
      lay.phys_out = next.data();
      lay.next_use = next_use[i].data();
      lay.target = home.data();
      // in place: the last part sends its qubits home, restore launches
      // fix the rest (ping-pong part 0 only prepares the next layout)
      lay.mode = (!pp && !no_restore && i + 1 == num_parts) ? LAYOUT_TARGET : LAYOUT_PRIORITY;
    }
    std::string e;
    const std::vector<int32_t>* gl = globals ? &(*globals)[i] : nullptr;
    int s = plan_part(n_local, dtype, tile_max, options, p.staged, p.num_staged, gates + p.gate_offset, p.num_gates,
                      plans[i], e, layout ? &lay : nullptr, gl && !gl->empty() ? gl->data() : nullptr,
                      gl ? (int)gl->size() : 0);
    if (s != HS_OK) {
      err = "part " + std::to_string(i) + ": " + e;
      return s;
    }
    plans[i].launch.in_buf = cur_buf;
    if (oop) cur_buf ^= 1;
    plans[i].launch.out_buf = cur_buf;
    plans[i].info.user_part = i;
    if (layout) {
      phys = next;
      for (int q = 0; q < n_local; ++q) inv[phys[q]] = q;
    }
  }
  if (pp && need_restore) {
    // stage qubits 0..hot-1 and the qubits on positions 0..hot-1: loads and
    // stores both run over 128 B lines; every other bit is a free bit
    std::vector<int32_t> st;
    for (int q = 0; q < hot; ++q) st.push_back(q);
    for (int pos = 0; pos < hot; ++pos)
      if (std::find(st.begin(), st.end(), inv[pos]) == st.end()) st.push_back(inv[pos]);
    std::sort(st.begin(), st.end());
    std::vector<int32_t> ident(n_local), next(phys);
    for (int q = 0; q < n_local; ++q) ident[q] = q;
    LayoutIO lay;
    lay.phys_in = phys.data();
    lay.inv_in = inv.data();
    lay.phys_out = next.data();
    lay.target = ident.data();
    lay.mode = LAYOUT_OOP;
    PartPlan pl;
    int s = plan_part(n_local, dtype, tile_max, options, st.data(), (int)st.size(), nullptr, 0, pl, err, &lay);
    if (s != HS_OK) return s;
    pl.info.restore = 1;
    pl.info.user_part = -1;
    pl.launch.in_buf = cur_buf;
    pl.launch.out_buf = cur_buf ^ 1;
    plans.push_back(pl);
    // the gate-free launch wrote natural order
    phys = next;
    for (int q = 0; q < n_local; ++q) inv[phys[q]] = q;
  }
  if (layout && !pp && !no_restore) {
    int s = plan_restore(n_local, dtype, tile_max, options, phys, plans, err);
    if (s != HS_OK) return s;
  }
  if (final_phys) final_phys->assign(phys.begin(), phys.begin() + n_local);  // identity once restored
  return HS_OK;
}

}  // namespace hs
