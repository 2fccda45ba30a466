// Part programs compiled to straight-line sm_100a kernels (NVRTC).
//
// The interpreter kernel (hs_kernels.cu) pays, for every gate, a dispatch
// (opcode/flag/target switch), matrix loads, and register moves that keep
// the 2^RB amplitudes in fixed registers across the dispatch loop. Here the
// planned instruction list of one part (the very same PartPlan the
// interpreter runs) is turned into CUDA C++ with everything resolved at
// compile time: shared-memory slots of every phase, register indices,
// control predicates, matrix entries (hex literals, which the compiler
// places in the constant bank and feeds straight into DFMA), and X-type
// exchanges on register bits, which become pure renamings (zero
// instructions). The CTA tile, phases and data movement are identical to
// the interpreter, so both paths are checked by the same parity tests.
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <cinttypes>
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <atomic>
#include <cstdlib>
#include <sys/stat.h>
#include <unistd.h>
#include <vector>

#include "hs_common.h"

namespace hs {

int jit_teams();

namespace {

uint32_t swz_host(uint32_t s, bool c128) {
  if (c128) return s ^ (((s >> 3) ^ (s >> 6) ^ (s >> 9) ^ (s >> 12)) & 7u);
  return s ^ (((s >> 4) ^ (s >> 8) ^ (s >> 12)) & 15u);
}

int sizeof_amp(bool c128) { return c128 ? 16 : 8; }

// tiles ahead the compiled kernels prefetch into L2 ($HISVSIM_L2_PREFETCH;
// default 0 = off: measured on c3, 1 / 2 / 3 / 5 tiles ahead cost 88.5 ->
// 97.8 / 98.5 / 115.9 / 126.8 ms, c2 5.26 -> 5.51 ms at 2)
// experiment switches read at code generation (part of the source, hence of
// the cubin cache key): HISVSIM_STORE_CS=1 stores the tile with st.global.cs
// (evict-first), HISVSIM_TILE_ORDER=chunk gives each CTA a contiguous range
// of tiles instead of the grid stride
bool env_on(const char* name, const char* value) {
  const char* e = std::getenv(name);
  return e && std::string(e) == value;
}

int l2_prefetch_ahead() {
  const char* e = std::getenv("HISVSIM_L2_PREFETCH");
  if (!e || !*e) return 0;
  return std::max(0, std::min(8, std::atoi(e)));
}

std::string lit_raw(double v, bool c128) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%a", v);
  std::string s(buf);
  if (!c128) s = "(float)(" + s + ")";
  return "(" + s + ")";
}

struct Gen {
  std::ostringstream o;
  bool c128;
  // two teams take turns on the FP64 pipe (HISVSIM_FP64_TOKEN=1): a team's
  // gates run between PP_ACQUIRE (after the phase's shared-memory loads) and
  // PP_RELEASE (before its stores), so one team exchanges while the other
  // computes instead of both doing the same thing at once
  bool token = false;
  int token_phases = 0;  // acquire / release pairs emitted per tile
  int token_threads = 0;  // both teams' threads
  int RB, T, n_local;
  int nreg;
  std::vector<int> var;  // register slot i -> variable index
  const char* R() const { return c128 ? "double" : "float"; }

  // FP64 literals of one kernel, deduplicated by magnitude: products and
  // factorisations of the same gate set give values a few ulps apart
  // (1/sqrt(2) came out in 12 spellings in one c2 part). ptxas keeps a
  // kernel's distinct constants in uniform registers while they fit (63 per
  // warp, 2 per FP64 value) and spills the rest to vector registers, which
  // makes the DFMA read three vector operands (the slow issue rate of
  // profiles/tools/fp64probe.cu). Values within 1e-14 relative of an earlier
  // one reuse it (negation is a free operand modifier); the change per gate
  // entry is ~50 ulps, far inside the 1e-10 tolerance.
  std::vector<double> pool;
  bool dedup = !env_on("HISVSIM_LIT_DEDUP", "0");  // "0": every literal as computed (A/B)
  std::string lit(double v, bool c) {
    const double a = std::fabs(v);
    if (dedup && a != 0.0 && a != 1.0) {
      for (double p : pool)
        if (std::fabs(a - p) <= 1e-14 * p) return lit_raw(v < 0 ? -p : p, c);
      pool.push_back(a);
    }
    return lit_raw(v, c);
  }

  std::string re(int i) { return "r" + std::to_string(var[i]); }
  std::string im(int i) { return "q" + std::to_string(var[i]); }

  // A diagonal's entry parity / control test over this thread's tile bits
  // (t) and the tile's global qubits (gw: the free index bits of the pass's
  // I_GLOBALS positions, one word per tile)
  std::string tparity(const Instr& in) const {
    const uint64_t gq = instr_gq(in);
    std::string e;
    if (in.qtid) e = "__popc(t & " + std::to_string(in.qtid) + "u)";
    if (gq) e += std::string(e.empty() ? "" : " + ") + "__popc(gw & " + std::to_string(gq) + "u)";
    return e.empty() ? std::string("false") : "(((" + e + ") & 1) != 0)";
  }
  std::string tcond(const Instr& in) const {
    const uint64_t gc = instr_gc(in);
    std::string e;
    if (in.ctid) e = "((t & " + std::to_string(in.ctid) + "u) == " + std::to_string(in.ctid) + "u)";
    if (gc) e += std::string(e.empty() ? "" : " && ") + "((gw & " + std::to_string(gc) + "u) == " + std::to_string(gc) + "u)";
    return e.empty() ? std::string("true") : "(" + e + ")";
  }

  // thread-dependent word tdep (tile location bits of this thread's amps)
  void emit_tdep(const char* name, const uint8_t* npos) {
    o << "    " << name << " = 0u";
    for (int m = 0; m < T - RB; ++m) o << " | (((tid >> " << m << ") & 1u) << " << (int)npos[m] << ")";
    o << ";\n";
  }
  std::vector<uint32_t> slot_xor(const uint8_t* rpos) {
    std::vector<uint32_t> u(nreg, 0);
    for (int i = 0; i < nreg; ++i)
      for (int k = 0; k < RB; ++k)
        if (i >> k & 1) u[i] ^= swz_host(1u << rpos[k], c128);
    return u;
  }
  // Cluster tiles: slot s lives in CTA s >> TC. A register's slot is this
  // CTA's own when the thread bits that carry the CTA rank (lowc..) map onto
  // the top tile locations TC.. and the register's own bits stay below TC;
  // own slots take plain shared-memory accesses, the rest go through DSMEM.
  bool carry = false;  // leave the part's scalar pending (Sr, Si) for a later launch
  bool cluster = false;
  int TC = 0, cl = 0, lowc = 0;
  bool rank_aligned(const uint8_t* npos) const {
    for (int r = 0; r < cl; ++r)
      if (npos[lowc + r] != TC + r) return false;
    return true;
  }
  bool reg_local(const uint8_t* npos, uint32_t u) const {
    return !cluster || (rank_aligned(npos) && (u >> TC) == 0);
  }
  bool phase_local(const uint8_t* rpos, const uint8_t* npos) {
    auto u = slot_xor(rpos);
    for (int i = 0; i < nreg; ++i)
      if (!reg_local(npos, u[i])) return false;
    return true;
  }
  // st ^ u with the swizzled low bits XORed and the rest added: st is zero
  // at the register locations and the swizzle only touches the low 3 (c128)
  // / 4 (c64) bits, so st ^ u == (st ^ (u & lo)) + (u & ~lo) and the added
  // part becomes the LDS/STS immediate offset (<= 2^lo distinct bases)
  std::string local_slot(uint32_t u) const {
    const uint32_t lo = c128 ? 7u : 15u;
    const std::string b = "(st ^ " + std::to_string(u & lo) + "u)";
    const std::string hi = std::to_string(u & ~lo) + "u";
    return cluster ? "(" + b + " & " + std::to_string((1u << TC) - 1) + "u) + " + hi : b + " + " + hi;
  }
  void load_regs(const uint8_t* rpos, const uint8_t* npos) {
    auto u = slot_xor(rpos);
    for (int i = 0; i < nreg; ++i) {
      if (!reg_local(npos, u[i]))
        o << "    CL_LD(st ^ " << u[i] << "u, " << re(i) << ", " << im(i) << ");\n";
      else
        o << "    { const C v = sm[" << local_slot(u[i]) << "]; " << re(i) << " = v.x; " << im(i) << " = v.y; }\n";
    }
  }
  void store_regs(const uint8_t* rpos, const uint8_t* npos) {
    auto u = slot_xor(rpos);
    for (int i = 0; i < nreg; ++i) {
      if (!reg_local(npos, u[i]))
        o << "    CL_ST(st ^ " << u[i] << "u, " << re(i) << ", " << im(i) << ");\n";
      else
        o << "    { C v; v.x = " << re(i) << "; v.y = " << im(i) << "; sm[" << local_slot(u[i]) << "] = v; }\n";
    }
  }
  void cmul_into(int i, const std::string& dr, const std::string& di) {
    o << "      { const " << R() << " x = " << re(i) << ", y = " << im(i) << "; " << re(i) << " = fma(x, " << dr
      << ", -y * " << di << "); " << im(i) << " = fma(x, " << di << ", y * " << dr << "); }\n";
    cat[1] += 4 * wgt; ops += 4 * wgt;
  }
  // multiply register i by a compile-time constant, exploiting 0 / +-1 parts
  void cmul_const(int i, double fr, double fi) {
    if (fr == 1.0 && fi == 0.0) return;
    if (fi == 0.0) {
      if (fr == -1.0) {
        o << "      " << re(i) << " = NEG(" << re(i) << "); " << im(i) << " = NEG(" << im(i) << ");\n";
        return;
      }
      o << "      " << re(i) << " *= " << lit(fr, c128) << "; " << im(i) << " *= " << lit(fr, c128) << ";\n";
      cat[2] += 2 * wgt; ops += 2 * wgt;
      return;
    }
    if (fr == 0.0) {  // (x + iy) * (i b) = -b y + i b x
      const std::string b = lit(fi, c128);
      o << "      { const " << R() << " x = " << re(i) << ", y = " << im(i) << "; ";
      if (fi == 1.0) o << re(i) << " = NEG(y); " << im(i) << " = x; }\n";
      else if (fi == -1.0) o << re(i) << " = y; " << im(i) << " = NEG(x); }\n";
      else {
        o << re(i) << " = -" << b << " * y; " << im(i) << " = " << b << " * x; }\n";
        cat[2] += 2 * wgt; ops += 2 * wgt;
      }
      return;
    }
    cmul_into(i, lit(fr, c128), lit(fi, c128));
  }

  // ---- the part's scalar. structure_2x2 and the diagonal-run folding
  // factor a constant s out of uncontrolled gates; every amplitude of the
  // state owes the product S of those constants, applied once before the
  // final store (folded into the last diagonal run when there is one).
  double Sr = 1.0, Si = 0.0;
  double ops = 0;   // FP64 instructions per thread per tile (control-weighted)
  double cat[5] = {0, 0, 0, 0, 0};  // of which: dense, diagonal apply, constant factors, mixed groups, scalar combine
  double wgt = 1;   // fraction of threads executing the current block
  bool scale_ok(double sr, double si) const {
    const double nr = Sr * sr - Si * si, ni = Sr * si + Si * sr;
    const double mag = std::hypot(nr, ni);
    // amplitudes stay far from overflow / underflow (complex64: 2^+-127)
    return mag > 0 && std::fabs(std::log2(mag)) < (c128 ? 300 : 48);
  }
  void push_scale(double sr, double si) {
    const double nr = Sr * sr - Si * si, ni = Sr * si + Si * sr;
    Sr = nr;
    Si = ni;
  }

  // one real output: sum_t coef[t] * src[t]; +-1 coefficients become adds
  std::string comb(const double coef[4], const std::string* src) {
    int start = -1;
    for (int t = 0; t < 4 && start < 0; ++t)
      if (coef[t] == 1.0) start = t;
    for (int t = 0; t < 4 && start < 0; ++t)
      if (coef[t] == -1.0) start = t;
    std::string e;
    if (start >= 0) e = (coef[start] == 1.0 ? "" : "-") + src[start];
    for (int t = 0; t < 4; ++t) {
      if (t == start || coef[t] == 0.0) continue;
      if (e.empty()) e = lit(coef[t], c128) + " * " + src[t];
      else if (coef[t] == 1.0) e = "(" + e + " + " + src[t] + ")";
      else if (coef[t] == -1.0) e = "(" + e + " - " + src[t] + ")";
      else e = "fma(" + lit(coef[t], c128) + ", " + src[t] + ", " + e + ")";
      cat[0] += wgt; ops += wgt;
    }
    if (start >= 0 && e == "-" + src[start]) return "NEG(" + src[start] + ")";  // a lone negation: sign bit
    return e.empty() ? std::string(c128 ? "0.0" : "0.0f") : e;
  }

  void dense(const Instr& in) {
    const bool plain = in.creg == 0 && in.ctid == 0;
    Mat2 M = structure_2x2(in.m, plain);
    if ((M.s[0] != 1.0 || M.s[1] != 0.0) && !scale_ok(M.s[0], M.s[1])) M = structure_2x2(in.m, false);
    push_scale(M.s[0], M.s[1]);
    const std::string src[4] = {"xr", "xi", "yr", "yi"};
    for (int i = 0; i < nreg; ++i) {
      if (i >> in.k & 1) continue;
      if ((uint32_t(i) & in.creg) != in.creg) continue;
      const int j = i | (1 << in.k);
      o << "      { const " << R() << " xr = " << re(i) << ", xi = " << im(i) << ", yr = " << re(j) << ", yi = "
        << im(j) << ";\n";
      const std::string dst[4] = {re(i), im(i), re(j), im(j)};
      for (int c = 0; c < 4; ++c) {
        double coef[4];
        component_coefs(M.m, c, coef);
        o << "        " << dst[c] << " = " << comb(coef, src) << ";\n";
      }
      o << "      }\n";
    }
  }

  void perm(const Instr& in, bool uniform) {
    for (int i = 0; i < nreg; ++i) {
      if (i >> in.k & 1) continue;
      if ((uint32_t(i) & in.creg) != in.creg) continue;
      const int j = i | (1 << in.k);
      if (uniform) {
        std::swap(var[i], var[j]);  // a renaming: no instruction
      } else {
        o << "      { const " << R() << " tr = " << re(i) << ", ti = " << im(i) << "; " << re(i) << " = " << re(j)
          << "; " << im(i) << " = " << im(j) << "; " << re(j) << " = tr; " << im(j) << " = ti; }\n";
      }
    }
  }

  // ---- folding of diagonal runs. Diagonal gates commute with each other, so
  // a run of them (up to the next non-diagonal instruction or phase change)
  // is applied as ONE complex factor per amplitude: gates that depend only
  // on register bits fold into a compile-time constant per register, gates
  // that depend only on thread bits fold into one runtime scalar per thread.
  // Gates mixing both are emitted as they come.
  std::vector<double> cre, cim;  // pending constant factor per register
  bool have_const = false, have_u = false;
  int u_id = 0;
  // pending mixed diagonals (register and thread bits, no controls): their
  // entry is d[parity(i & kreg) ^ parity(t & qtid)]. Grouped by register
  // mask, a group's factor for register i is F_g[parity(i & kreg)], where
  // F_g[0] / F_g[1] are per-thread products of d[tp] / d[!tp] over the
  // group's gates (no per-amplitude work); register i then costs one complex
  // multiply per extra group plus one to apply, instead of one per gate.
  std::vector<Instr> mixed;
  int m_id = 0;

  void reset_pending() {
    cre.assign(nreg, 1.0);
    cim.assign(nreg, 0.0);
    have_const = have_u = false;
    mixed.clear();
  }
  // mixed run: per-thread group factors, then one factor per register
  void flush_mixed() {
    std::vector<uint32_t> masks;
    for (const Instr& in : mixed) {
      const uint32_t kreg = (in.flags & F_PARITY) ? in.rpos[0] : (1u << in.k);
      if (std::find(masks.begin(), masks.end(), kreg) == masks.end()) masks.push_back(kreg);
    }
    ++m_id;
    const std::string T = R(), M = "m" + std::to_string(m_id) + "_";
    o << "    {\n";
    for (size_t gi = 0; gi < masks.size(); ++gi) {
      const std::string a = M + std::to_string(gi);
      o << "      " << T << " " << a << "r0, " << a << "i0, " << a << "r1, " << a << "i1;\n";
      bool first = true;
      for (const Instr& in : mixed) {
        const uint32_t kreg = (in.flags & F_PARITY) ? in.rpos[0] : (1u << in.k);
        if (kreg != masks[gi]) continue;
        const std::string d0r = lit(in.m[0], c128), d0i = lit(in.m[1], c128);
        const std::string d1r = lit(in.m[2], c128), d1i = lit(in.m[3], c128);
        o << "      { const bool tp = " << tparity(in) << ";\n";
        o << "        const " << T << " ar = tp ? " << d1r << " : " << d0r << ", ai = tp ? " << d1i << " : " << d0i
          << ", br = tp ? " << d0r << " : " << d1r << ", bi = tp ? " << d0i << " : " << d1i << ";\n";
        if (first) {
          o << "        " << a << "r0 = ar; " << a << "i0 = ai; " << a << "r1 = br; " << a << "i1 = bi; }\n";
          first = false;
        } else {
          ops += 8.0;  // per thread, not per amplitude (ops counts a thread's instructions)
          o << "        { const " << T << " x = " << a << "r0, y = " << a << "i0; " << a << "r0 = x * ar - y * ai; "
            << a << "i0 = x * ai + y * ar; }\n";
          o << "        { const " << T << " x = " << a << "r1, y = " << a << "i1; " << a << "r1 = x * br - y * bi; "
            << a << "i1 = x * bi + y * br; } }\n";
        }
      }
    }
    // the thread-uniform scalar joins group 0 (per thread, not per amplitude)
    if (have_u) {
      ops += 8.0;
      const std::string a = M + "0", ur = "ur" + std::to_string(u_id), ui = "ui" + std::to_string(u_id);
      for (int b = 0; b < 2; ++b) {
        const std::string r = a + "r" + std::to_string(b), i = a + "i" + std::to_string(b);
        o << "      { const " << T << " x = " << r << ", y = " << i << "; " << r << " = x * " << ur << " - y * " << ui
          << "; " << i << " = x * " << ui << " + y * " << ur << "; }\n";
      }
    }
    // registers sharing a factor (the same group parities) back to back:
    // the factor of a parity signature is built once per thread (G - 1
    // complex multiplies per distinct signature, not per register)
    std::vector<int> reg_order(nreg);
    for (int i = 0; i < nreg; ++i) reg_order[i] = i;
    auto signature = [&](int i) {
      int sig = 0;
      for (size_t gi = 0; gi < masks.size(); ++gi) sig |= (__builtin_popcount(uint32_t(i) & masks[gi]) & 1) << gi;
      return sig;
    };
    // registers with the same signature and the same constant factor (the
    // run's register-only diagonals) share one per-thread factor: the
    // constant is folded into it once per thread, not multiplied into every
    // register on its own
    auto key_less = [&](int x, int y) {
      if (signature(x) != signature(y)) return signature(x) < signature(y);
      if (cre[x] != cre[y]) return cre[x] < cre[y];
      return cim[x] < cim[y];
    };
    std::stable_sort(reg_order.begin(), reg_order.end(), key_less);
    int cur_sig = -1;
    double cur_r = 0, cur_i = 0;
    bool open_sig = false, open_const = false;
    for (int i : reg_order) {
      const int sig = signature(i);
      const bool new_sig = sig != cur_sig;
      const bool new_const = new_sig || cre[i] != cur_r || cim[i] != cur_i;
      if (new_const && open_const) { o << "      }\n"; open_const = false; }
      if (new_sig) {
        if (open_sig) o << "      }\n";
        cur_sig = sig;
        open_sig = true;
        o << "      {";
        for (size_t gi = 0; gi < masks.size(); ++gi) {
          const int par = sig >> gi & 1;
          const std::string r = M + std::to_string(gi) + "r" + std::to_string(par);
          const std::string im_ = M + std::to_string(gi) + "i" + std::to_string(par);
          if (gi == 0) {
            o << " " << T << " fr = " << r << ", fi = " << im_ << ";";
          } else {
            o << " { const " << T << " x = fr, y = fi; fr = x * " << r << " - y * " << im_ << "; fi = x * " << im_
              << " + y * " << r << "; }";
            cat[3] += 4.0; ops += 4.0;  // per thread, not per amplitude
          }
        }
        o << "\n";
      }
      if (new_const) {
        cur_r = cre[i];
        cur_i = cim[i];
        open_const = true;
        o << "      {";
        if (cur_r == 1.0 && cur_i == 0.0) {
          o << " const " << T << " gr = fr, gi = fi;\n";
        } else {  // (fr + i fi) * constant, once per thread
          const std::string cr = lit(cur_r, c128), ci = lit(cur_i, c128);
          o << " const " << T << " gr = fr * " << cr << " - fi * " << ci << ", gi = fr * " << ci << " + fi * " << cr
            << ";\n";
          cat[4] += 4.0; ops += 4.0;  // per thread
        }
      }
      o << "  ";
      cmul_into(i, "gr", "gi");
    }
    if (open_const) o << "      }\n";
    if (open_sig) o << "      }\n";
    o << "    }\n";
  }
  // final: fold the part's scalar S into the run and apply it (no
  // normalisation); otherwise the most common factor of the run is pulled
  // out into S so the registers carrying it cost nothing
  // keep_u: the instruction that forces the flush acts on register bits
  // only (dense / X-type gates): a pending per-thread scalar alone commutes
  // with it (it scales all of the thread's registers alike) and waits for
  // the next flush, which applies it for free, or the phase's end
  void flush(bool final = false, bool keep_u = false) {
    if (keep_u && !final && have_u && !have_const && mixed.empty()) return;
    if (final && (Sr != 1.0 || Si != 0.0)) {
      for (int i = 0; i < nreg; ++i) {
        const double nr = cre[i] * Sr - cim[i] * Si, ni = cre[i] * Si + cim[i] * Sr;
        cre[i] = nr;
        cim[i] = ni;
      }
      have_const = true;
      Sr = 1.0;
      Si = 0.0;
    }
    if (!have_const && !have_u && mixed.empty()) return;
    if (have_const && !final) {
      int best = -1, best_n = 0;
      for (int i = 0; i < nreg; ++i) {
        int n = 0;
        for (int j = 0; j < nreg; ++j) n += cre[j] == cre[i] && cim[j] == cim[i];
        if (n > best_n) { best_n = n; best = i; }
      }
      const double fr = cre[best], fi = cim[best];
      const double n2 = fr * fr + fi * fi;
      if (!(fr == 1.0 && fi == 0.0) && n2 > 0 && scale_ok(fr, fi)) {
        for (int i = 0; i < nreg; ++i) {
          if (cre[i] == fr && cim[i] == fi) { cre[i] = 1.0; cim[i] = 0.0; continue; }
          double nr = (cre[i] * fr + cim[i] * fi) / n2, ni = (cim[i] * fr - cre[i] * fi) / n2;
          if (std::fabs(ni) < 2e-15) ni = 0;
          if (std::fabs(nr) < 2e-15) nr = 0;
          if (ni == 0 && std::fabs(nr - 1) < 2e-15) nr = 1;
          if (ni == 0 && std::fabs(nr + 1) < 2e-15) nr = -1;
          if (nr == 0 && std::fabs(ni - 1) < 2e-15) ni = 1;
          if (nr == 0 && std::fabs(ni + 1) < 2e-15) ni = -1;
          cre[i] = nr;
          cim[i] = ni;
        }
        push_scale(fr, fi);
      }
    }
    if (!mixed.empty()) {
      flush_mixed();
      reset_pending();
      return;
    }
    o << "    {\n";
    if (!have_u) {
      for (int i = 0; i < nreg; ++i) cmul_const(i, cre[i], cim[i]);
    } else {
      // registers with the same constant share one per-thread factor
      // (constant x scalar, once per thread per distinct constant)
      const std::string ur = "ur" + std::to_string(u_id), ui = "ui" + std::to_string(u_id);
      std::vector<int> order(nreg);
      for (int i = 0; i < nreg; ++i) order[i] = i;
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        return cre[x] != cre[y] ? cre[x] < cre[y] : cim[x] < cim[y];
      });
      bool open = false;
      double cr_ = 0, ci_ = 0;
      for (int i : order) {
        if (!open || cre[i] != cr_ || cim[i] != ci_) {
          if (open) o << "      }\n";
          open = true;
          cr_ = cre[i];
          ci_ = cim[i];
          if (cr_ == 1.0 && ci_ == 0.0) {
            o << "      { const " << R() << " fr = " << ur << ", fi = " << ui << ";\n";
          } else {
            o << "      { const " << R() << " fr = fma(" << lit(cr_, c128) << ", " << ur << ", -" << lit(ci_, c128)
              << " * " << ui << "), fi = fma(" << lit(cr_, c128) << ", " << ui << ", " << lit(ci_, c128) << " * "
              << ur << ");\n";
            cat[4] += 4.0; ops += 4.0;  // per thread
          }
        }
        o << "  ";
        cmul_into(i, "fr", "fi");
      }
      if (open) o << "      }\n";
    }
    o << "    }\n";
    reset_pending();
  }
  // returns true if the instruction was folded into the pending run
  bool fold_diag(const Instr& in) {
    const bool parity = in.flags & F_PARITY;
    const uint32_t kreg = parity ? in.rpos[0] : (in.k == K_NONE ? 0u : (1u << in.k));
    const bool tdep = in.qtid != 0 || in.ctid != 0 || instr_gq(in) != 0 || instr_gc(in) != 0;
    const bool rdep = kreg != 0 || in.creg != 0;
    const double d0r = in.m[0], d0i = in.m[1], d1r = in.m[2], d1i = in.m[3];
    if (!tdep) {
      for (int i = 0; i < nreg; ++i) {
        if ((uint32_t(i) & in.creg) != in.creg) continue;
        const bool one = __builtin_popcount(uint32_t(i) & kreg) & 1;
        const double fr = one ? d1r : d0r, fi = one ? d1i : d0i;
        const double nr = cre[i] * fr - cim[i] * fi, ni = cre[i] * fi + cim[i] * fr;
        cre[i] = nr;
        cim[i] = ni;
      }
      have_const = true;
      return true;
    }
    if (rdep) {
      // controlled ones, and sign flips (integer XORs, no FP64), are applied as they come
      if (in.creg != 0 || in.ctid != 0 || instr_gc(in) != 0 || cluster || (in.flags & F_SIGN)) return false;
      mixed.push_back(in);
      return true;
    }
    // uniform per thread: one scalar factor, selected by this thread's bits
    if (!have_u) {
      ++u_id;
      o << "    " << R() << " ur" << u_id << " = 1, ui" << u_id << " = 0;\n";
      have_u = true;
    }
    const std::string ur = "ur" + std::to_string(u_id), ui = "ui" + std::to_string(u_id);
    o << "    { const bool tp = " << tparity(in) << ";\n";
    const std::string cond = tcond(in);
    o << "      if (" << cond << ") { const " << R() << " fr = tp ? " << lit(d1r, c128) << " : " << lit(d0r, c128)
      << ", fi = tp ? " << lit(d1i, c128) << " : " << lit(d0i, c128) << "; const " << R() << " a = " << ur << ", b = "
      << ui << "; " << ur << " = a * fr - b * fi; " << ui << " = a * fi + b * fr; } }\n";
    ops += 4;
    return true;
  }

  void diag(const Instr& in) {
    const std::string d0r = lit(in.m[0], c128), d0i = lit(in.m[1], c128);
    const std::string d1r = lit(in.m[2], c128), d1i = lit(in.m[3], c128);
    const bool sign = in.flags & F_SIGN, d0one = in.flags & F_D0_ONE, d1one = in.flags & F_D1_ONE;
    const bool parity = in.flags & F_PARITY;
    const uint32_t kreg = parity ? in.rpos[0] : (in.k == K_NONE ? 0u : (1u << in.k));
    const bool tbits = in.qtid != 0 || instr_gq(in) != 0;
    if (tbits) o << "      const bool tp = " << tparity(in) << ";\n";
    for (int i = 0; i < nreg; ++i) {
      if ((uint32_t(i) & in.creg) != in.creg) continue;
      const bool rp = __builtin_popcount(uint32_t(i) & kreg) & 1;
      // entry index = rp ^ tp
      if (!tbits) {
        const bool one = rp;
        if (one) {
          if (sign) o << "      " << re(i) << " = NEG(" << re(i) << "); " << im(i) << " = NEG(" << im(i) << ");\n";
          else if (!d1one) cmul_const(i, in.m[2], in.m[3]);
        } else if (!d0one) {
          cmul_const(i, in.m[0], in.m[1]);
        }
        continue;
      }
      const std::string one = rp ? "!tp" : "tp";
      if (sign) {
        // sign flip on the integer pipe: XOR the sign bit under a per-thread mask
        o << "      { const SM m_ = (" << one << ") ? SIGN_BIT : SM(0); " << re(i) << " = XSGN(" << re(i) << ", m_); "
          << im(i) << " = XSGN(" << im(i) << ", m_); }\n";
      } else {
        o << "      { const " << R() << " dr = " << one << " ? " << d1r << " : " << d0r << ", di = " << one << " ? "
          << d1i << " : " << d0i << ";\n  ";
        cmul_into(i, "dr", "di");
        o << "      }\n";
      }
    }
  }
};

// The part's program on one tile: register declarations, phases (shared
// memory exchanges separated by `sync`), gates, the part's scalar, and the
// final write of the registers into the tile's store order (ending in `sync`)
void emit_program(Gen& g, const PartPlan& pl, const char* sync, double* fp64_per_amp,
                  const char* local_sync = "__syncthreads();", const char* after_last_load = nullptr) {
  std::ostringstream& o = g.o;
  const Instr* last_phase = nullptr;
  for (const Instr& in : pl.prog)
    if (in.op == I_PHASE) last_phase = &in;
  // cluster tiles: an exchange whose writes and reads all stay in this CTA's
  // slots (for every CTA alike: the mapping is the same) needs only a CTA
  // barrier; otherwise the cluster barrier
  auto xsync = [&](const uint8_t* r0, const uint8_t* n0, const uint8_t* r1, const uint8_t* n1) -> std::string {
    if (g.cluster && g.phase_local(r0, n0) && g.phase_local(r1, n1)) return local_sync;
    return sync;
  };
  o << "    " << g.R() << " ";
  for (int i = 0; i < g.nreg; ++i) o << (i ? ", " : "") << "r" << i << ", q" << i;
  o << ";\n    unsigned t, st;\n";
  // the turns: a team takes its turn before a phase's shared-memory loads
  // (memory operations stay behind the barrier) and passes it on once the
  // phase's arithmetic is done. ptxas moves arithmetic freely across a
  // barrier, so the passing barrier's id depends on every amplitude register
  // through a value it cannot know is zero (zero_: high bits of ntiles)
  auto take_turn = [&]() { o << "    PP_ACQUIRE();\n"; };
  auto pass_turn = [&]() {
    o << "    { unsigned h_ = 0u;";
    for (int i = 0; i < g.nreg; ++i) {
      if (g.c128) o << " h_ ^= (unsigned)__double2hiint(r" << i << ") ^ (unsigned)__double2hiint(q" << i << ");";
      else o << " h_ ^= __float_as_uint(r" << i << ") ^ __float_as_uint(q" << i << ");";
    }
    o << "\n      asm volatile(\"bar.arrive %0, " << g.token_threads << ";\" :: \"r\"(3u + (team ^ 1u) + (h_ & zero_)) : \"memory\"); }\n";
  };
  const Instr* cur = nullptr;
  g.reset_pending();
  for (const Instr& in : pl.prog) {
    if (in.op == I_GLOBALS) continue;  // the kernel's gw word (jit_source)
    if (in.op == I_DIAG && g.fold_diag(in)) continue;
    if (in.op != I_DIAG) g.flush(false, in.op == I_DENSE || in.op == I_PERM);  // apply the pending run first
    if (in.op == I_PHASE) {
      if (cur) {
        if (g.token) pass_turn();
        g.store_regs(cur->rpos, cur->npos);
        o << "    " << xsync(cur->rpos, cur->npos, in.rpos, in.npos) << "\n";
      }
      g.emit_tdep("t", in.npos);
      o << "    st = swz(t);\n";
      if (g.token) {
        take_turn();
        ++g.token_phases;
      }
      g.load_regs(in.rpos, in.npos);
      if (&in == last_phase && after_last_load) o << "    " << after_last_load << "\n";
      cur = &in;
      continue;
    }
    const bool ctl_t = in.ctid != 0 || instr_gc(in) != 0;
    if (ctl_t) o << "    if (" << g.tcond(in) << ") {\n";
    else o << "    {\n";
    g.wgt = 1.0 / double(1u << __builtin_popcount(in.ctid));
    if (in.op == I_DENSE) g.dense(in);
    else if (in.op == I_PERM) g.perm(in, !ctl_t);
    else g.diag(in);
    g.wgt = 1.0;
    o << "    }\n";
  }
  // pending diagonal run + the part's scalar: the scalar is global, so it is
  // carried to the program's last launch unless it grows large
  const bool apply = !g.carry || std::fabs(std::log2(std::hypot(g.Sr, g.Si))) > (g.c128 ? 200 : 24);
  g.flush(apply);
  if (g.token && cur) pass_turn();
  if (fp64_per_amp) *fp64_per_amp = g.ops / g.nreg;
  o << "    // fp64_instr_per_amp " << g.ops / g.nreg << " (dense " << g.cat[0] / g.nreg << ", diagonal apply "
    << g.cat[1] / g.nreg << ", constants " << g.cat[2] / g.nreg << ", mixed groups " << g.cat[3] / g.nreg
    << ", scalar combine " << g.cat[4] / g.nreg << ")\n";
  if (pl.launch.direct_store) return;  // the caller stores the registers to HBM
  // the final write goes to the store order; the read-out after it is local
  const std::string fs = xsync(cur->rpos, cur->npos, pl.launch.fin_rpos, pl.launch.fin_npos);
  if (pl.launch.fin_sync) o << "    " << fs << "\n";
  g.emit_tdep("t", pl.launch.fin_npos);
  o << "    st = swz(t);\n";
  g.store_regs(pl.launch.fin_rpos, pl.launch.fin_npos);
  o << "    " << (g.cluster && g.phase_local(pl.launch.fin_rpos, pl.launch.fin_npos) ? local_sync : sync)
    << "\n";
}

std::string jit_source(const PartPlan& pl, int dtype, int n_local, double* fp64_per_amp = nullptr,
                       double* carry_scale = nullptr, bool last = true) {
  Gen g;
  if (carry_scale) {  // in: scalar owed by earlier launches; out: what this one leaves pending
    g.carry = !last;
    g.Sr = carry_scale[0];
    g.Si = carry_scale[1];
  }
  g.c128 = dtype == HS_C128;
  g.RB = pl.launch.RB;
  g.T = pl.launch.T;
  g.n_local = n_local;
  g.nreg = 1 << g.RB;
  g.var.resize(g.nreg);
  for (int i = 0; i < g.nreg; ++i) g.var[i] = i;
  // cluster tiles (parts wider than one CTA's tile): 2^cl CTAs, one per SM,
  // each holding the 2^TC slots s with s >> TC == its rank
  const int cl = pl.launch.cluster_log, C_SIZE = 1 << cl;
  const int T = g.T, RB = g.RB, TC = T - cl, low = TC - RB, NT = 1 << low;
  if (cl > 0) {
    g.cluster = true;
    g.TC = TC;
    g.cl = cl;
    g.lowc = low;
  }
  const uint32_t lmask = (1u << TC) - 1;
  const char* C = g.c128 ? "double2" : "float2";
  const int amp = g.c128 ? 16 : 8;
  std::ostringstream& o = g.o;
  o << "typedef " << C << " C;\n";
  if (g.c128)
    o << "typedef unsigned long long SM;\n#define SIGN_BIT 0x8000000000000000ull\n"
      << "__device__ __forceinline__ double XSGN(double x, SM m) { return __longlong_as_double(__double_as_longlong(x) ^ (long long)m); }\n";
  else
    o << "typedef unsigned SM;\n#define SIGN_BIT 0x80000000u\n"
      << "__device__ __forceinline__ float XSGN(float x, SM m) { return __uint_as_float(__float_as_uint(x) ^ m); }\n";
  // a sign flip the compiler cannot turn back into an FP64 negation
  if (g.c128)
    o << "__device__ __forceinline__ double NEG(double x) { double r; asm(\"{ .reg .b32 lo_, hi_; mov.b64 {lo_, hi_}, %1; "
         "xor.b32 hi_, hi_, 0x80000000; mov.b64 %0, {lo_, hi_}; }\" : \"=d\"(r) : \"d\"(x)); return r; }\n";
  else
    o << "__device__ __forceinline__ float NEG(float x) { float r; asm(\"xor.b32 %0, %1, 0x80000000;\" : \"=f\"(r) : \"f\"(x)); "
         "return r; }\n";
  o << "__device__ __forceinline__ unsigned swz(unsigned s) { return s ^ "
    << (g.c128 ? "(((s >> 3) ^ (s >> 6) ^ (s >> 9) ^ (s >> 12)) & 7u)" : "(((s >> 4) ^ (s >> 8) ^ (s >> 12)) & 15u)")
    << "; }\n";
  // One CTA per SM: two teams of NT threads each run the part on their own
  // tiles (team 0 takes the CTA's even tiles, team 1 the odd ones) in one of
  // three shared-memory tile buffers; the third buffer receives the tile
  // after next while both teams compute. Tile i of the CTA lives in buffer
  // i % 3; whichever team finishes tile i refills that buffer with tile
  // i + 3 (cp.async, completion counted on the buffer's mbarrier by
  // cp.async.mbarrier.arrive.noinc), so loads stay in flight across tiles.
  // Teams synchronise with named barriers (1 + team). Cluster tiles: team t
  // of every CTA of the cluster works on the same tile; an exchange that
  // crosses CTAs ends in a team-wide cluster barrier (TEAM_CSYNC: a named
  // barrier, then one thread release-arrives on that team's mbarrier in
  // every CTA, then all acquire-wait on their own; two mbarriers alternate
  // so consecutive uses never share a phase).
  const int tile_bytes = amp << TC;
  if (NT >= 32)
    o << "#define TEAM_SYNC() asm volatile(\"bar.sync %0, " << NT << ";\" :: \"r\"(bar_id) : \"memory\")\n";
  else  // tiny tiles: both teams share warp 0
    o << "#define TEAM_SYNC() __syncwarp(" << ((1ull << NT) - 1) << "u << (team * " << NT << "u))\n";
  if (cl > 0) {
    const char* V = g.c128 ? "v2.f64" : "v2.f32";
    const char* RC = g.c128 ? "d" : "f";
    o << "__device__ __forceinline__ unsigned cl_addr(unsigned sbase, unsigned sl) {\n  unsigned ra;\n"
      << "  asm volatile(\"mapa.shared::cluster.u32 %0, %1, %2;\" : \"=r\"(ra) : \"r\"(sbase + (sl & " << lmask
      << "u) * " << amp << "u), \"r\"(sl >> " << TC << "));\n  return ra;\n}\n";
    o << "#define CL_ADDR(sl) cl_addr(sbase, (sl))\n";
    o << "#define CL_ST(sl, x, y) asm volatile(\"st.shared::cluster." << V << " [%0], {%1, %2};\" :: \"r\"(CL_ADDR(sl)), \""
      << RC << "\"(x), \"" << RC << "\"(y) : \"memory\")\n";
    o << "#define CL_LD(sl, x, y) asm volatile(\"ld.shared::cluster." << V << " {%0, %1}, [%2];\" : \"=" << RC << "\"(x), \"="
      << RC << "\"(y) : \"r\"(CL_ADDR(sl)) : \"memory\")\n";
    o << "__device__ __forceinline__ void team_csync(unsigned tb, unsigned& k, unsigned bar_id, unsigned tid0) {\n"
      << "  asm volatile(\"bar.sync %0, " << NT << ";\" :: \"r\"(bar_id) : \"memory\");\n"
      << "  const unsigned mb = tb + (k & 1u) * 8u;\n"
      << "  if (tid0 == 0) {\n"
      << "    for (unsigned q = 0; q < " << C_SIZE << "u; ++q) {\n"
      << "      unsigned ra;\n"
      << "      asm volatile(\"mapa.shared::cluster.u32 %0, %1, %2;\" : \"=r\"(ra) : \"r\"(mb), \"r\"(q));\n"
      << "      asm volatile(\"mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\" :: \"r\"(ra) : \"memory\");\n"
      << "    }\n  }\n"
      << "  const unsigned par = (k >> 1) & 1u;\n  unsigned done = 0;\n"
      << "  while (!done) asm volatile(\"{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
         "selp.u32 %0, 1, 0, p; }\" : \"=r\"(done) : \"r\"(mb), \"r\"(par) : \"memory\");\n"
      << "  ++k;\n" << (NT >= 32 ? "  __syncwarp();\n" : "") << "}\n";
    o << "#define TEAM_CSYNC() team_csync(tb_team, csync_k, bar_id, tid0)\n";
  }
  // teams per CTA ($HISVSIM_TEAMS): 2 (default) alternate tiles; 1 keeps two
  // tile loads in flight while the single team computes (cluster tiles: 2)
  const int TEAMS = cl > 0 ? 2 : jit_teams();
  o << "extern \"C\" __global__ void __launch_bounds__(" << TEAMS * NT << ", 1) hs_jit_part(C* psi, C* psi_out, long long ntiles) {\n";
  o << "  extern __shared__ __align__(128) unsigned char smem_raw[];\n";
  o << "  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw + " << 3 * tile_bytes << ");\n";
  o << "  volatile int* issued = reinterpret_cast<volatile int*>(smem_raw + " << 3 * tile_bytes + 32 << ");\n";
  o << "  const unsigned team = threadIdx.x >> " << low << ";\n";
  o << "  const unsigned tid0 = threadIdx.x & " << (NT - 1) << "u;\n";
  o << "  const unsigned bar_id = 1u + team;\n";
  if (cl > 0) {
    o << "  unsigned long long* tbar = reinterpret_cast<unsigned long long*>(smem_raw + " << 3 * tile_bytes + 64 << ");\n";
    o << "  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_raw);\n";
    o << "  unsigned rank, cid, ncl;\n";
    o << "  asm(\"mov.u32 %0, %%cluster_ctarank;\" : \"=r\"(rank));\n";
    o << "  asm(\"mov.u32 %0, %%clusterid.x;\" : \"=r\"(cid));\n";
    o << "  asm(\"mov.u32 %0, %%nclusterid.x;\" : \"=r\"(ncl));\n";
    o << "  const unsigned tb_team = (unsigned)__cvta_generic_to_shared(&tbar[2 * team]);\n";
    o << "  unsigned csync_k = 0;\n";
    o << "  const unsigned sw_rank = swz(rank << " << TC << ") & " << lmask << "u;\n";
  } else {
    o << "  const unsigned rank = 0, cid = blockIdx.x, ncl = gridDim.x, sw_rank = 0;\n";
  }
  if (cl == 0 && env_on("HISVSIM_TILE_ORDER", "chunk")) {
    o << "  const long long per_cta = (ntiles + ncl - 1) / ncl;\n";
    o << "#define TILE(i) ((long long)cid * per_cta + (i))\n";
    o << "#define TILE_OK(i, t) ((i) < per_cta && (t) < ntiles)\n";
  } else {
    o << "#define TILE(i) ((long long)cid + (i) * (long long)ncl)\n";
    o << "#define TILE_OK(i, t) ((t) < ntiles)\n";
  }
  o << "  if (threadIdx.x == 0) {\n";
  o << "    for (int b = 0; b < 3; ++b) asm volatile(\"mbarrier.init.shared::cta.b64 [%0], " << NT
    << ";\" :: \"r\"((unsigned)__cvta_generic_to_shared(&full[b])) : \"memory\");\n";
  if (cl > 0)
    o << "    for (int b = 0; b < 4; ++b) asm volatile(\"mbarrier.init.shared::cta.b64 [%0], " << C_SIZE
      << ";\" :: \"r\"((unsigned)__cvta_generic_to_shared(&tbar[b])) : \"memory\");\n";
  o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
  o << "    for (int b = 0; b < 3; ++b) issued[b] = 0;\n  }\n";
  if (cl > 0)  // every CTA's barriers exist before any peer arrives on them
    o << "  asm volatile(\"barrier.cluster.arrive.release.aligned;\\n\\tbarrier.cluster.wait.acquire.aligned;\" ::: \"memory\");\n";
  else
    o << "  __syncthreads();\n";
  // canonical load order of this CTA's slots: s = tid0 + (j << low) + (rank << TC)
  auto dep = [&](const uint8_t* pos, const char* what, int from, int cnt) {
    std::string e = "0ull";
    for (int b = 0; b < cnt; ++b)
      e += " | ((unsigned long long)((" + std::string(what) + " >> " + std::to_string(b) + ") & 1u) << " +
           std::to_string((int)pos[from + b]) + ")";
    return e;
  };
  o << "  const unsigned long long ga_tid = " << dep(pl.launch.tpos, "tid0", 0, low) << " | "
    << dep(pl.launch.tpos, "rank", TC, cl) << ";\n";
  o << "  const unsigned sw_tid = swz(tid0) ^ sw_rank;\n";
  // tile -> global offset of its slot 0 (zero bits inserted at the tile positions)
  o << "  auto tile_base = [&](long long tt) -> unsigned long long {\n";
  o << "    const unsigned long long row = (unsigned long long)tt >> " << (n_local - T) << ";\n";
  o << "    unsigned long long f = (unsigned long long)tt & " << ((1ull << (n_local - T)) - 1) << "ull;\n";
  for (int b = 0; b < T; ++b) {
    int p = pl.launch.tpos[b];
    o << "    { const unsigned long long lo = f & " << ((1ull << p) - 1) << "ull; f = ((f ^ lo) << 1) | lo; }\n";
  }
  o << "    return (row << " << n_local << ") | f | ga_tid;\n  };\n";
  const bool oop = pl.launch.oop != 0;
  if (oop) {  // out of place: the same tile under the next layout
    o << "  const unsigned long long go_tid = " << dep(pl.launch.opos, "tid0", 0, low) << " | "
      << dep(pl.launch.opos, "rank", TC, cl) << ";\n";
    o << "  auto out_base = [&](long long tt) -> unsigned long long {\n";
    o << "    const unsigned long long f = (unsigned long long)tt;\n";
    o << "    return ((f >> " << (n_local - T) << ") << " << n_local << ") | go_tid";
    for (int j = 0; j < n_local - T; ++j) o << "\n      | (((f >> " << j << ") & 1ull) << " << (int)pl.launch.fpos[j] << ")";
    o << ";\n  };\n";
  }
  auto ohi_of = [&](int j) {
    uint64_t hi = 0;
    for (int k = 0; k < RB; ++k)
      if (j >> k & 1) hi |= 1ull << (oop ? pl.launch.opos[low + k] : pl.launch.tpos[low + k]);
    return hi;
  };
  auto hi_of = [&](int j) {
    uint64_t hi = 0;
    for (int k = 0; k < RB; ++k)
      if (j >> k & 1) hi |= 1ull << pl.launch.tpos[low + k];
    return hi;
  };
  // issue the loads of CTA tile i into buffer i % 3 (this thread's share)
  o << "  auto issue = [&](long long i) {\n";
  o << "    const long long tt = TILE(i);\n";
  o << "    if (!TILE_OK(i, tt)) return;\n";
  o << "    const unsigned long long base = tile_base(tt);\n";
  o << "    const int b = (int)(i % 3);\n";
  o << "    const unsigned sb = (unsigned)__cvta_generic_to_shared(smem_raw) + b * " << tile_bytes << "u;\n";
  for (int j = 0; j < g.nreg; ++j) {
    const uint32_t sx = swz_host(uint32_t(j) << low, g.c128) & lmask;
    o << "    asm volatile(\"cp.async." << (g.c128 ? "cg" : "ca") << ".shared.global [%0], [%1], "
      << amp << ";\" :: \"r\"(sb + (sw_tid ^ " << sx << "u) * " << amp
      << "u), \"l\"(psi + (base | " << hi_of(j) << "ull)) : \"memory\");\n";
  }
  o << "    asm volatile(\"cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\" :: \"r\"((unsigned)__cvta_generic_to_shared(&full[b])) : \"memory\");\n";
  o << "    if (tid0 == 0) issued[b] = (int)(i / 3);\n";
  // L2 prefetch of the tile `ahead` loads later: the three tile buffers keep
  // at most one tile (64 KB) of reads in flight per SM, below what HBM
  // latency x per-SM bandwidth needs; lines prefetched into L2 a few tiles
  // early make those cp.async loads L2 hits. One prefetch per 128 B line:
  // only threads / registers whose tile bits on storage positions 0..2 are
  // zero issue one.
  const int ahead = l2_prefetch_ahead();
  if (ahead > 0 && cl == 0) {
    uint32_t lane_mask = 0, reg_mask = 0;
    for (int k = 0; k < low; ++k)
      if (pl.launch.tpos[k] < 3) lane_mask |= 1u << k;
    for (int k = 0; k < RB; ++k)
      if (pl.launch.tpos[low + k] < 3) reg_mask |= 1u << k;
    o << "    { const long long tp = TILE(i + " << ahead << ");\n";
    o << "      if (TILE_OK(i + " << ahead << ", tp) && (tid0 & " << lane_mask << "u) == 0u) {\n";
    o << "        const unsigned long long pb = tile_base(tp);\n";
    for (int j = 0; j < g.nreg; ++j) {
      if (uint32_t(j) & reg_mask) continue;
      o << "        asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(psi + (pb | " << hi_of(j) << "ull)));\n";
    }
    o << "      } }\n";
  }
  o << "  };\n";
  // HISVSIM_FP64_TOKEN: "1" every two-team launch, "auto" only launches with
  // little arithmetic (at most TOKEN_AUTO_GATES gate instructions per tile:
  // memory-bound passes and gate-free layout launches), else off. Measured on
  // c3 (ms per launch, turns / no turns): FP64-heavy launches 10.6 / 8.7,
  // 14.6 / 12.5 (the turn serialises the loads of one team with the
  // arithmetic of the other); the memory-bound last launch 5.43 / 6.20
  int gate_instrs = 0;
  for (const Instr& in : pl.prog) gate_instrs += in.op == I_DENSE || in.op == I_PERM || in.op == I_DIAG;
  constexpr int TOKEN_AUTO_GATES = 10;
  const char* tok_env = std::getenv("HISVSIM_FP64_TOKEN");
  const std::string tok = tok_env && *tok_env ? tok_env : "auto";  // default: auto; "0" off; "1" every launch
  g.token = TEAMS == 2 && cl == 0 && NT >= 32 &&
            (tok == "1" || (tok == "auto" && gate_instrs <= TOKEN_AUTO_GATES));
  g.token_threads = 2 * NT;
  if (g.token) {
    // named barriers 3 + team: a team waits on its own, the other team's
    // release arrives on it (2 * NT participants); team 1 hands team 0 the
    // first turn
    o << "#define PP_ACQUIRE() asm volatile(\"bar.sync %0, " << 2 * NT << ";\" :: \"r\"(3u + team) : \"memory\")\n";
    o << "#define PP_RELEASE() asm volatile(\"bar.arrive %0, " << 2 * NT << ";\" :: \"r\"(3u + (team ^ 1u)) : \"memory\")\n";
    o << "  const unsigned zero_ = (unsigned)((unsigned long long)ntiles >> 62);\n";
    o << "  if (team == 1) PP_RELEASE();\n";
  }
  if (TEAMS == 2) {
    o << "  issue(team);\n  if (team == 0) issue(2);\n";
    o << "  for (long long i = team;; i += 2) {\n";
  } else {
    o << "  issue(0);\n  issue(1);\n  issue(2);\n";
    o << "  for (long long i = 0;; ++i) {\n";
  }
  o << "    const long long tt = TILE(i);\n";
  o << "    if (!TILE_OK(i, tt)) break;\n";
  o << "    const unsigned long long base = tile_base(tt);\n";
  for (const Instr& in : pl.prog) {  // the tile's global qubits (free index bits of the input)
    if (in.op != I_GLOBALS) continue;
    const uint8_t* gp = reinterpret_cast<const uint8_t*>(in.m);
    o << "    const unsigned gw = 0u";
    for (int j = 0; j < in.k; ++j) o << " | ((unsigned)((base >> " << (int)gp[j] << ") & 1ull) << " << j << ")";
    o << ";\n";
  }
  o << "    unsigned tid = tid0 | (rank << " << low << "); asm volatile(\"\" : \"+r\"(tid));  // keep phase addresses in the loop\n";
  o << "    const int b = (int)(i % 3);\n";
  o << "    C* sm = reinterpret_cast<C*>(smem_raw + b * " << tile_bytes << ");\n";
  if (cl > 0) o << "    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);\n";
  // Fill k = i / 3 of buffer b. This team can get here before the other
  // team has even issued fill k (it is still on tile i - 3), and a parity
  // wait cannot tell phase k from phase k - 2. The producer publishes the
  // fill number it issued (issued[b]); once it reads k, phase k is the
  // newest phase that can complete and the parity wait is unambiguous.
  o << "    { const long long k = i / 3;\n";
  o << "      if (k > 0) while (issued[b] < (int)k) __nanosleep(20);\n";
  o << "      const unsigned mb = (unsigned)__cvta_generic_to_shared(&full[b]); const unsigned par = (unsigned)(k & 1);\n";
  o << "      unsigned done = 0;\n";
  o << "      while (!done) asm volatile(\"{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\" : \"=r\"(done) : \"r\"(mb), \"r\"(par) : \"memory\"); }\n";
  // Reconverge the warp after the data-dependent wait loops: without it
  // ptxas treats the rest of the tile as divergent code and keeps the gate
  // constants in vector registers (three-vector-operand DFMAs at ~2/3 of the
  // issue rate, profiles/tools/fp64reuse.cu) instead of uniform registers.
  // A warp belongs to one team unless the teams share warp 0 (tiny tiles).
  const bool reconverge = NT >= 32 && !env_on("HISVSIM_SYNCWARP", "0");  // "0": A/B without
  if (reconverge) o << "    __syncwarp();\n";
  if (cl > 0) {  // the first phase reads other CTAs' slots: their loads must be in
    const Instr* first = nullptr;
    for (const Instr& in : pl.prog)
      if (in.op == I_PHASE) { first = &in; break; }
    if (!(first && g.phase_local(first->rpos, first->npos))) o << "    TEAM_CSYNC();\n";
  }
  const bool direct = pl.launch.direct_store && cl == 0;
  // direct stores: the buffer is free once the last phase has loaded its
  // registers, so its refill (tile i + 3) overlaps the last phase's gates
  emit_program(g, pl, cl > 0 ? "TEAM_CSYNC();" : "TEAM_SYNC();", fp64_per_amp, "TEAM_SYNC();",
               direct ? (reconverge ? "TEAM_SYNC(); issue(i + 3); __syncwarp();" : "TEAM_SYNC(); issue(i + 3);") : nullptr);
  const FuseSwitch& fz = pl.fuse;
  if (oop) o << "    const unsigned long long obase = out_base(tt);\n";
  // fused layout switch: every amplitude goes to the rank that owns it after
  // the switch - the one picked by its output index's bits at the outgoing
  // qubits' positions (per tile when those are free bits, per register or
  // lane when they are tile bits) - at the same index with those bits
  // replaced by this rank's slot (FSTORE)
  if (oop && fz.on) {
    uint64_t pam = 0, slotbits = 0;
    for (int b = 0; b < fz.c; ++b) {
      pam |= 1ull << fz.pa[b];
      if (fz.slot >> b & 1) slotbits |= 1ull << fz.pa[b];
    }
    std::ostringstream sel;
    sel << "unsigned k_ = 0u;";
    for (int b = 0; b < fz.c; ++b) sel << " k_ |= (unsigned)((x_ >> " << fz.pa[b] << ") & 1ull) << " << b << ";";
    std::ostringstream ptr;
    for (int k = 0; k < (1 << fz.c); ++k)
      ptr << (k + 1 < (1 << fz.c) ? "k_ == " + std::to_string(k) + "u ? " : "") << "0x" << std::hex << fz.out_ptr[k]
          << std::dec << "ull" << (k + 1 < (1 << fz.c) ? " : " : "");
    o << "#define FSTORE(X, V) do { const unsigned long long x_ = (X); " << sel.str()
      << " reinterpret_cast<C*>(" << ptr.str() << ")[(x_ & ~" << pam << "ull) | " << slotbits
      << "ull] = (V); } while (0)\n";
  }
  const bool fstore = oop && fz.on;
  if (direct) {
    // store slot bit r sits at output position pos[r]; lanes 0..2 carry slot
    // bits 0..2, so each warp instruction writes whole 128 B lines
    const uint8_t* pos = oop ? pl.launch.opos : pl.launch.tpos;
    o << "    const unsigned long long dbase = " << (oop ? "(obase ^ go_tid)" : "(base ^ ga_tid)") << " | 0ull";
    for (int m = 0; m < T - RB; ++m)
      o << " | ((unsigned long long)((tid >> " << m << ") & 1u) << " << (int)pos[pl.launch.fin_npos[m]] << ")";
    o << ";\n";
    for (int i = 0; i < g.nreg; ++i) {
      uint64_t off = 0;
      for (int k = 0; k < RB; ++k)
        if (i >> k & 1) off |= 1ull << pos[pl.launch.fin_rpos[k]];
      if (fstore)
      o << "    { C v; v.x = " << g.re(i) << "; v.y = " << g.im(i) << "; FSTORE(dbase | " << off << "ull, v); }\n";
    else if (env_on("HISVSIM_STORE_CS", "1"))
      o << "    { C v; v.x = " << g.re(i) << "; v.y = " << g.im(i) << "; __stcs(&" << (oop ? "psi_out" : "psi")
        << "[dbase | " << off << "ull], v); }\n";
    else
      o << "    { C v; v.x = " << g.re(i) << "; v.y = " << g.im(i) << "; " << (oop ? "psi_out" : "psi") << "[dbase | "
        << off << "ull] = v; }\n";
    }
    o << "  }\n";
    if (g.token) {
      // the turns alternate strictly: the team that runs out of tiles first
      // keeps passing the turn while the other finishes its extra tile
      o << "  { long long cnt = 0; while (TILE_OK(cnt, TILE(cnt))) ++cnt;\n"
        << "    const long long mine = (cnt + 1 - (long long)team) / 2, other = (cnt + (long long)team) / 2;\n"
        << "    for (long long x = mine; x < other; ++x)\n"
        << "      for (int ph = 0; ph < " << g.token_phases << "; ++ph) { PP_ACQUIRE(); PP_RELEASE(); } }\n";
    }
    o << "}\n";
  } else {
    for (int j = 0; j < g.nreg; ++j) {
      const uint32_t sx = swz_host(uint32_t(j) << low, g.c128) & lmask;
      const std::string dst = oop ? std::string("psi_out[obase | ") : std::string("psi[base | ");
      if (fstore)
        o << "    FSTORE(obase | " << ohi_of(j) << "ull, sm[sw_tid ^ " << sx << "u]);\n";
      else if (env_on("HISVSIM_STORE_CS", "1"))
        o << "    __stcs(&" << dst << ohi_of(j) << "ull], sm[sw_tid ^ " << sx << "u]);\n";
      else
        o << "    " << dst << ohi_of(j) << "ull] = sm[sw_tid ^ " << sx << "u];\n";
    }
    o << "    TEAM_SYNC();\n";  // the buffer is free: refill it with tile i + 3
    o << "    issue(i + 3);\n";
    o << "  }\n";
    if (g.token) {
      // the turns alternate strictly: the team that runs out of tiles first
      // keeps passing the turn while the other finishes its extra tile
      o << "  { long long cnt = 0; while (TILE_OK(cnt, TILE(cnt))) ++cnt;\n"
        << "    const long long mine = (cnt + 1 - (long long)team) / 2, other = (cnt + (long long)team) / 2;\n"
        << "    for (long long x = mine; x < other; ++x)\n"
        << "      for (int ph = 0; ph < " << g.token_phases << "; ++ph) { PP_ACQUIRE(); PP_RELEASE(); } }\n";
    }
    o << "}\n";
  }
  if (carry_scale) {
    carry_scale[0] = g.Sr;
    carry_scale[1] = g.Si;
  }
  return o.str();
}

std::mutex g_cache_mu;
std::map<std::string, void*> g_cache;  // source -> kernel handle

// ---- on-disk cubin cache. A one-shot execute_hierarchical plans and
// compiles its parts in every new process; NVRTC is ~0.5-1 s per circuit
// (parallel over parts) while the planner takes tens of ms. Cubins are kept
// under $HISVSIM_CACHE_DIR (default $XDG_CACHE_HOME/hisvsim or
// ~/.cache/hisvsim; "off" disables), keyed by a 64-bit FNV-1a hash of the
// generated source, the NVRTC options and the NVRTC version; the entry also
// stores the full source, compared on load, so a hash collision is a miss.
// (line info: ncu maps the compiled passes' SASS back to the generated source)
const char* kNvrtcOpts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device", "--generate-line-info"};

std::string cache_dir() {
  const char* d = std::getenv("HISVSIM_CACHE_DIR");
  if (d && *d) return std::string(d) == "off" ? std::string() : std::string(d);
  if (const char* x = std::getenv("XDG_CACHE_HOME"); x && *x) return std::string(x) + "/hisvsim";
  if (const char* h = std::getenv("HOME"); h && *h) return std::string(h) + "/.cache/hisvsim";
  return std::string();
}

std::string cache_key(const std::string& src) {
  int major = 0, minor = 0;
  nvrtcVersion(&major, &minor);
  std::string all = src;
  for (const char* o : kNvrtcOpts) all += std::string("\n//opt ") + o;
  all += "\n//nvrtc " + std::to_string(major) + "." + std::to_string(minor);
  uint64_t h = 1469598103934665603ull;
  for (unsigned char ch : all) { h ^= ch; h *= 1099511628211ull; }
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%016" PRIx64, h);
  return buf;
}

// entry: uint64 source length, source bytes, cubin bytes
bool cache_load(const std::string& dir, const std::string& key, const std::string& src, std::vector<char>& cubin) {
  if (dir.empty()) return false;
  FILE* f = std::fopen((dir + "/" + key + ".cubin").c_str(), "rb");
  if (!f) return false;
  bool ok = false;
  uint64_t n = 0;
  if (std::fread(&n, sizeof(n), 1, f) == 1 && n == src.size()) {
    std::string s(n, '\0');
    if (std::fread(&s[0], 1, n, f) == n && s == src) {
      std::vector<char> body;
      char buf[1 << 16];
      size_t got;
      while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) body.insert(body.end(), buf, buf + got);
      if (!body.empty()) { cubin.swap(body); ok = true; }
    }
  }
  std::fclose(f);
  return ok;
}

void cache_store(const std::string& dir, const std::string& key, const std::string& src, const std::vector<char>& cubin) {
  if (dir.empty()) return;
  // mkdir -p (one level below an existing parent is the common case)
  for (size_t i = 1; i <= dir.size(); ++i)
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
  char tmp_name[64];
  std::snprintf(tmp_name, sizeof(tmp_name), ".tmp.%d.%zx", (int)getpid(),
                std::hash<std::thread::id>()(std::this_thread::get_id()));
  const std::string tmp = dir + "/" + key + tmp_name, dst = dir + "/" + key + ".cubin";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;
  const uint64_t n = src.size();
  bool ok = std::fwrite(&n, sizeof(n), 1, f) == 1 && std::fwrite(src.data(), 1, n, f) == n &&
            std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
  ok = (std::fclose(f) == 0) && ok;
  if (ok) std::rename(tmp.c_str(), dst.c_str());  // atomic: readers see whole entries only
  else std::remove(tmp.c_str());
}

std::atomic<int> g_disk_hits{0}, g_compiles{0};

int nvrtc_compile(const std::string& src, std::vector<char>& cubin, std::string& err);

int compile_one(const std::string& src, void** kernel, std::string& err) {
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(src);
    if (it != g_cache.end()) { *kernel = it->second; return HS_OK; }
  }
  const std::string dir = cache_dir();
  const std::string key = dir.empty() ? std::string() : cache_key(src);
  std::vector<char> cubin;
  if (cache_load(dir, key, src, cubin)) {
    ++g_disk_hits;
  } else {
    int s = nvrtc_compile(src, cubin, err);
    if (s != HS_OK) return s;
    ++g_compiles;
    cache_store(dir, key, src, cubin);
  }
  cudaLibrary_t lib;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) { err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e); return HS_ERR_CUDA; }
  cudaKernel_t k;
  e = cudaLibraryGetKernel(&k, lib, "hs_jit_part");
  if (e != cudaSuccess) { err = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e); return HS_ERR_CUDA; }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache[src] = (void*)k;
  *kernel = (void*)k;
  return HS_OK;
}

int nvrtc_compile(const std::string& src, std::vector<char>& cubin, std::string& err) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "hs_part.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    err = "nvrtcCreateProgram failed";
    return HS_ERR_UNSUPPORTED;
  }
  nvrtcResult r = nvrtcCompileProgram(prog, (int)(sizeof(kNvrtcOpts) / sizeof(kNvrtcOpts[0])), kNvrtcOpts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    err = "NVRTC: " + log.substr(0, 2000);
    return HS_ERR_UNSUPPORTED;
  }
  size_t sz = 0;
  nvrtcGetCUBINSize(prog, &sz);
  cubin.resize(sz);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  return HS_OK;
}

}  // namespace

int jit_compile_program(std::vector<PartPlan>& plans, int dtype, int n_local, int device, int smem_optin,
                        std::string& err) {
  const size_t n = plans.size();
  std::vector<std::string> srcs(n);
  std::vector<double> fp64(n, 0.0);
  // the structured-gate scalars multiply into one global factor, applied by
  // the last launch (runs of a program's launches must be complete, in order)
  double scale[2] = {1.0, 0.0};
  for (size_t i = 0; i < n; ++i) {
    plans[i].carry_in[0] = scale[0];
    plans[i].carry_in[1] = scale[1];
    plans[i].last = i + 1 == n;
    srcs[i] = jit_source(plans[i], dtype, n_local, &fp64[i], scale, i + 1 == n);
  }
  std::vector<int> status(n, HS_OK);
  std::vector<std::string> errs(n);
  unsigned hw = std::thread::hardware_concurrency();
  const size_t workers = std::max<size_t>(1, std::min<size_t>(n, hw ? hw : 4));
  std::vector<std::thread> pool;
  for (size_t w = 0; w < workers; ++w)
    pool.emplace_back([&, w]() {
      cudaSetDevice(device);
      for (size_t i = w; i < n; i += workers) status[i] = compile_one(srcs[i], &plans[i].jit, errs[i]);
    });
  for (auto& t : pool) t.join();
  for (size_t i = 0; i < n; ++i) {
    if (status[i] != HS_OK) {
      err = "part " + std::to_string(i) + ": " + errs[i];
      for (auto& p : plans) p.jit = nullptr;
      return status[i];
    }
    cudaFuncSetAttribute((const void*)plans[i].jit, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
    plans[i].info.fp64_instr_per_amp = (float)fp64[i];
  }
  return HS_OK;
}

std::string jit_source_for(const PartPlan& pl, int dtype, int n_local) { return jit_source(pl, dtype, n_local); }
double jit_fp64_per_amp(const PartPlan& pl, int dtype, int n_local) {
  double f = 0.0;
  jit_source(pl, dtype, n_local, &f);
  return f;
}

int jit_recompile(PartPlan& pl, int dtype, int n_local, int device, int smem_optin, std::string& err) {
  double scale[2] = {pl.carry_in[0], pl.carry_in[1]};
  double fp64 = 0.0;
  const std::string src = jit_source(pl, dtype, n_local, &fp64, scale, pl.last);
  cudaSetDevice(device);
  void* k = nullptr;
  const int s = compile_one(src, &k, err);
  if (s != HS_OK) return s;
  cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  pl.jit = k;
  return HS_OK;
}

std::string hs_cache_dir() { return cache_dir(); }

int jit_teams() {
  const char* e = std::getenv("HISVSIM_TEAMS");
  return (e && std::atoi(e) == 1) ? 1 : 2;
}

void jit_cache_stats(int* disk_hits, int* compiles) {
  if (disk_hits) *disk_hits = g_disk_hits.load();
  if (compiles) *compiles = g_compiles.load();
}

}  // namespace hs
