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
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "hs_common.h"

namespace hs {

namespace {

uint32_t swz_host(uint32_t s, bool c128) {
  if (c128) return s ^ (((s >> 3) ^ (s >> 6) ^ (s >> 9) ^ (s >> 12)) & 7u);
  return s ^ (((s >> 4) ^ (s >> 8) ^ (s >> 12)) & 15u);
}

std::string lit(double v, bool c128) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%a", v);
  std::string s(buf);
  if (!c128) s = "(float)(" + s + ")";
  return "(" + s + ")";
}

struct Gen {
  std::ostringstream o;
  bool c128;
  int RB, T, n_local;
  int nreg;
  std::vector<int> var;  // register slot i -> variable index
  const char* R() const { return c128 ? "double" : "float"; }

  std::string re(int i) { return "r" + std::to_string(var[i]); }
  std::string im(int i) { return "q" + std::to_string(var[i]); }

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
  void load_regs(const uint8_t* rpos) {
    auto u = slot_xor(rpos);
    for (int i = 0; i < nreg; ++i)
      o << "    { const C v = sm[st ^ " << u[i] << "u]; " << re(i) << " = v.x; " << im(i) << " = v.y; }\n";
  }
  void store_regs(const uint8_t* rpos) {
    auto u = slot_xor(rpos);
    for (int i = 0; i < nreg; ++i)
      o << "    { C v; v.x = " << re(i) << "; v.y = " << im(i) << "; sm[st ^ " << u[i] << "u] = v; }\n";
  }
  void cmul_into(int i, const std::string& dr, const std::string& di) {
    o << "      { const " << R() << " x = " << re(i) << ", y = " << im(i) << "; " << re(i) << " = fma(x, " << dr
      << ", -y * " << di << "); " << im(i) << " = fma(x, " << di << ", y * " << dr << "); }\n";
  }

  void dense(const Instr& in) {
    const double* m = in.m;
    const bool real = in.flags & F_REAL;
    std::string M[8];
    for (int q = 0; q < 8; ++q) M[q] = lit(m[q], c128);
    for (int i = 0; i < nreg; ++i) {
      if (i >> in.k & 1) continue;
      if ((uint32_t(i) & in.creg) != in.creg) continue;
      const int j = i | (1 << in.k);
      o << "      { const " << R() << " xr = " << re(i) << ", xi = " << im(i) << ", yr = " << re(j) << ", yi = "
        << im(j) << ";\n";
      if (real) {
        o << "        " << re(i) << " = fma(" << M[0] << ", xr, " << M[2] << " * yr); " << im(i) << " = fma(" << M[0]
          << ", xi, " << M[2] << " * yi);\n";
        o << "        " << re(j) << " = fma(" << M[4] << ", xr, " << M[6] << " * yr); " << im(j) << " = fma(" << M[4]
          << ", xi, " << M[6] << " * yi); }\n";
      } else {
        auto out = [&](const std::string& dst_r, const std::string& dst_i, int a, int b) {
          // (ma + i mb) * x + (mc + i md) * y with (a, b) = entries of x, y
          o << "        " << dst_r << " = fma(" << M[a] << ", xr, fma(-" << M[a + 1] << ", xi, fma(" << M[b]
            << ", yr, -" << M[b + 1] << " * yi)));\n";
          o << "        " << dst_i << " = fma(" << M[a] << ", xi, fma(" << M[a + 1] << ", xr, fma(" << M[b]
            << ", yi, " << M[b + 1] << " * yr)));\n";
        };
        out(re(i), im(i), 0, 2);
        out(re(j), im(j), 4, 6);
        o << "      }\n";
      }
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

  void reset_pending() {
    cre.assign(nreg, 1.0);
    cim.assign(nreg, 0.0);
    have_const = have_u = false;
  }
  void flush() {
    if (!have_const && !have_u) return;
    o << "    {\n";
    for (int i = 0; i < nreg; ++i) {
      const bool unit = cre[i] == 1.0 && cim[i] == 0.0;
      if (!have_u) {
        if (unit) continue;
        if (cre[i] == -1.0 && cim[i] == 0.0) {
          o << "      " << re(i) << " = -" << re(i) << "; " << im(i) << " = -" << im(i) << ";\n";
          continue;
        }
        cmul_into(i, lit(cre[i], c128), lit(cim[i], c128));
        continue;
      }
      const std::string ur = "ur" + std::to_string(u_id), ui = "ui" + std::to_string(u_id);
      if (unit) {
        cmul_into(i, ur, ui);
      } else {
        o << "      { const " << R() << " fr = fma(" << lit(cre[i], c128) << ", " << ur << ", -" << lit(cim[i], c128)
          << " * " << ui << "), fi = fma(" << lit(cre[i], c128) << ", " << ui << ", " << lit(cim[i], c128) << " * "
          << ur << ");\n  ";
        cmul_into(i, "fr", "fi");
        o << "      }\n";
      }
    }
    o << "    }\n";
    reset_pending();
  }
  // returns true if the instruction was folded into the pending run
  bool fold_diag(const Instr& in) {
    const bool parity = in.flags & F_PARITY;
    const uint32_t kreg = parity ? in.rpos[0] : (in.k == K_NONE ? 0u : (1u << in.k));
    const bool tdep = in.qtid != 0 || in.ctid != 0;
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
    if (rdep) return false;
    // uniform per thread: one scalar factor, selected by this thread's bits
    if (!have_u) {
      ++u_id;
      o << "    " << R() << " ur" << u_id << " = 1, ui" << u_id << " = 0;\n";
      have_u = true;
    }
    const std::string ur = "ur" + std::to_string(u_id), ui = "ui" + std::to_string(u_id);
    o << "    { const bool tp = (__popc(t & " << in.qtid << "u) & 1) != 0;\n";
    std::string cond = in.ctid ? "((t & " + std::to_string(in.ctid) + "u) == " + std::to_string(in.ctid) + "u)" : "true";
    o << "      if (" << cond << ") { const " << R() << " fr = tp ? " << lit(d1r, c128) << " : " << lit(d0r, c128)
      << ", fi = tp ? " << lit(d1i, c128) << " : " << lit(d0i, c128) << "; const " << R() << " a = " << ur << ", b = "
      << ui << "; " << ur << " = a * fr - b * fi; " << ui << " = a * fi + b * fr; } }\n";
    return true;
  }

  void diag(const Instr& in) {
    const std::string d0r = lit(in.m[0], c128), d0i = lit(in.m[1], c128);
    const std::string d1r = lit(in.m[2], c128), d1i = lit(in.m[3], c128);
    const bool sign = in.flags & F_SIGN, d0one = in.flags & F_D0_ONE, d1one = in.flags & F_D1_ONE;
    const bool parity = in.flags & F_PARITY;
    const uint32_t kreg = parity ? in.rpos[0] : (in.k == K_NONE ? 0u : (1u << in.k));
    const bool tbits = in.qtid != 0;
    if (tbits) o << "      const bool tp = (__popc(t & " << in.qtid << "u) & 1) != 0;\n";
    for (int i = 0; i < nreg; ++i) {
      if ((uint32_t(i) & in.creg) != in.creg) continue;
      const bool rp = __builtin_popcount(uint32_t(i) & kreg) & 1;
      // entry index = rp ^ tp
      if (!tbits) {
        const bool one = rp;
        if (one) {
          if (sign) o << "      " << re(i) << " = -" << re(i) << "; " << im(i) << " = -" << im(i) << ";\n";
          else if (!d1one) cmul_into(i, d1r, d1i);
        } else if (!d0one) {
          cmul_into(i, d0r, d0i);
        }
        continue;
      }
      const std::string one = rp ? "!tp" : "tp";
      if (sign) {
        o << "      if (" << one << ") { " << re(i) << " = -" << re(i) << "; " << im(i) << " = -" << im(i) << "; }\n";
      } else {
        o << "      { const " << R() << " dr = " << one << " ? " << d1r << " : " << d0r << ", di = " << one << " ? "
          << d1i << " : " << d0i << ";\n  ";
        cmul_into(i, "dr", "di");
        o << "      }\n";
      }
    }
  }
};

std::string jit_source(const PartPlan& pl, int dtype, int n_local) {
  Gen g;
  g.c128 = dtype == HS_C128;
  g.RB = pl.launch.RB;
  g.T = pl.launch.T;
  g.n_local = n_local;
  g.nreg = 1 << g.RB;
  g.var.resize(g.nreg);
  for (int i = 0; i < g.nreg; ++i) g.var[i] = i;
  const int T = g.T, RB = g.RB, low = T - RB, NT = 1 << low;
  const char* C = g.c128 ? "double2" : "float2";
  std::ostringstream& o = g.o;
  o << "typedef " << C << " C;\n";
  o << "__device__ __forceinline__ unsigned swz(unsigned s) { return s ^ "
    << (g.c128 ? "(((s >> 3) ^ (s >> 6) ^ (s >> 9) ^ (s >> 12)) & 7u)" : "(((s >> 4) ^ (s >> 8) ^ (s >> 12)) & 15u)")
    << "; }\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << NT << ", 2) hs_jit_part(C* __restrict__ psi, long long ntiles) {\n";
  o << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n  C* sm = reinterpret_cast<C*>(smem_raw);\n";
  o << "  const unsigned tid = threadIdx.x;\n";
  // canonical load order: slot s = tid + (j << low); global offset of tid part
  o << "  unsigned long long ga_tid = 0ull";
  for (int b = 0; b < low; ++b) o << " | ((unsigned long long)((tid >> " << b << ") & 1u) << " << (int)pl.launch.tpos[b] << ")";
  o << ";\n  const unsigned sw_tid = swz(tid);\n";
  uint64_t tile_mask = 0;
  for (int b = 0; b < T; ++b) tile_mask |= 1ull << pl.launch.tpos[b];
  o << "  for (long long tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {\n";
  o << "    const unsigned long long row = (unsigned long long)tt >> " << (n_local - T) << ";\n";
  o << "    unsigned long long f = (unsigned long long)tt & " << ((1ull << (n_local - T)) - 1) << "ull;\n";
  for (int b = 0; b < T; ++b) {
    int p = pl.launch.tpos[b];
    o << "    { const unsigned long long lo = f & " << ((1ull << p) - 1) << "ull; f = ((f ^ lo) << 1) | lo; }\n";
  }
  o << "    const unsigned long long base = (row << " << n_local << ") | f | ga_tid;\n";
  auto io = [&](bool load) {
    for (int j = 0; j < g.nreg; ++j) {
      uint64_t hi = 0;
      for (int k = 0; k < RB; ++k)
        if (j >> k & 1) hi |= 1ull << pl.launch.tpos[low + k];
      const uint32_t sx = swz_host(uint32_t(j) << low, g.c128);
      if (load)
        o << "    { const unsigned s = (unsigned)__cvta_generic_to_shared(&sm[sw_tid ^ " << sx << "u]);\n"
          << "      asm volatile(\"cp.async." << (g.c128 ? "cg" : "ca") << ".shared.global [%0], [%1], "
          << (g.c128 ? 16 : 8) << ";\" :: \"r\"(s), \"l\"(psi + (base | " << hi << "ull))); }\n";
      else
        o << "    psi[base | " << hi << "ull] = sm[sw_tid ^ " << sx << "u];\n";
    }
  };
  io(true);
  o << "    asm volatile(\"cp.async.commit_group;\\ncp.async.wait_group 0;\" ::: \"memory\");\n";
  o << "    __syncthreads();\n";
  o << "    " << g.R() << " ";
  for (int i = 0; i < g.nreg; ++i) o << (i ? ", " : "") << "r" << i << ", q" << i;
  o << ";\n    unsigned t, st;\n";
  const Instr* cur = nullptr;
  g.reset_pending();
  for (const Instr& in : pl.prog) {
    if (in.op == I_DIAG && g.fold_diag(in)) continue;
    if (in.op != I_DIAG) g.flush();  // a non-diagonal step: apply the pending run first
    if (in.op == I_PHASE) {
      if (cur) {
        g.store_regs(cur->rpos);
        o << "    __syncthreads();\n";
      }
      g.emit_tdep("t", in.npos);
      o << "    st = swz(t);\n";
      g.load_regs(in.rpos);
      cur = &in;
      continue;
    }
    const bool ctl_t = in.ctid != 0;
    if (ctl_t) o << "    if ((t & " << in.ctid << "u) == " << in.ctid << "u) {\n";
    else o << "    {\n";
    if (in.op == I_DENSE) g.dense(in);
    else if (in.op == I_PERM) g.perm(in, !ctl_t);
    else g.diag(in);
    o << "    }\n";
  }
  g.flush();
  if (pl.launch.fin_sync) o << "    __syncthreads();\n";
  g.emit_tdep("t", pl.launch.fin_npos);
  o << "    st = swz(t);\n";
  g.store_regs(pl.launch.fin_rpos);
  o << "    __syncthreads();\n";
  io(false);
  o << "    __syncthreads();\n  }\n}\n";
  return o.str();
}

std::mutex g_cache_mu;
std::map<std::string, void*> g_cache;  // source -> kernel handle

int compile_one(const std::string& src, void** kernel, std::string& err) {
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(src);
    if (it != g_cache.end()) { *kernel = it->second; return HS_OK; }
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "hs_part.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    err = "nvrtcCreateProgram failed";
    return HS_ERR_UNSUPPORTED;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device"};
  nvrtcResult r = nvrtcCompileProgram(prog, 3, opts);
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
  std::vector<char> cubin(sz);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
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

}  // namespace

int jit_compile_program(std::vector<PartPlan>& plans, int dtype, int n_local, int device, int smem_optin,
                        std::string& err) {
  const size_t n = plans.size();
  std::vector<std::string> srcs(n);
  for (size_t i = 0; i < n; ++i) srcs[i] = jit_source(plans[i], dtype, n_local);
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
  }
  return HS_OK;
}

std::string jit_source_for(const PartPlan& pl, int dtype, int n_local) { return jit_source(pl, dtype, n_local); }

}  // namespace hs
