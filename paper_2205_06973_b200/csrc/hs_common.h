// Internal definitions shared by the planner (host C++) and the part kernels.
#pragma once
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hisvsim.h"

namespace hs {

// Device instruction opcodes of a part program.
enum : uint16_t {
  I_PHASE = 1,  // write registers back (previous map), barrier, load with a new map
  I_DENSE = 2,  // 2x2 on register bit k, predicated on controls
  I_PERM = 3,   // X-type exchange on register bit k, predicated on controls
  I_DIAG = 4,   // diag(d0, d1) on a target bit (register k or tid-mask), predicated
  // compiled passes only (first instruction of a program that has them): the
  // physical positions of the pass's global qubits - qubits some diagonal
  // gate acts on that are not staged; their values are the tile's free index
  // bits. k = count, the positions are bytes of m[] (up to 64).
  I_GLOBALS = 5,
};

// DIAG flags
// F_PARITY (DIAG): the entry index is the parity of the register bits in
// rpos[0] (mask over the register index) and the thread bits in qtid
enum : uint8_t { F_D0_ONE = 1, F_D1_ONE = 2, F_SIGN = 4, F_PLAIN = 8, F_REAL = 16, F_PARITY = 32 };

constexpr uint8_t K_NONE = 0xFF;
constexpr int MAX_RB = 4;       // register bits per thread
constexpr int MAX_TILE = 13;    // tile bits the single-CTA kernels support
constexpr int MAX_CLUSTER_LOG = 2;  // compiled parts: tiles over clusters of up to 4 CTAs
constexpr int MAX_NPOS = 12;    // non-register tile bits (T - RB)

// One device instruction, 96 bytes. Location bits are positions inside the
// CTA tile (0..T-1) in the current storage labelling.
struct alignas(16) Instr {
  uint16_t op;
  uint8_t k;       // register index of the target (DENSE/PERM/DIAG) or K_NONE
  uint8_t flags;
  uint32_t creg;   // controls that are register bits: mask over register index
  uint32_t ctid;   // controls that are thread bits: mask over tile location bits
  uint32_t qtid;   // DIAG target as a tile-location mask when not a register bit
  uint8_t rpos[MAX_RB];    // PHASE: location of register bit k
  uint8_t npos[MAX_NPOS];  // PHASE: location of thread-index bit m
  double m[8];     // DENSE: m00 m01 m10 m11 (re, im); DIAG: d0, d1
};
static_assert(sizeof(Instr) == 96, "Instr layout");
// DIAG instructions on global qubits keep two more masks in m[4] / m[5]
// (raw bits; a DIAG uses only m[0..3]): gq = global qubits in the entry's
// parity, gc = global controls (bit j = the program's I_GLOBALS entry j).
inline uint64_t instr_gq(const Instr& in) {
  if (in.op != I_DIAG) return 0;
  uint64_t v;
  std::memcpy(&v, &in.m[4], 8);
  return v;
}
inline uint64_t instr_gc(const Instr& in) {
  if (in.op != I_DIAG) return 0;
  uint64_t v;
  std::memcpy(&v, &in.m[5], 8);
  return v;
}
inline void instr_set_global(Instr& in, uint64_t gq, uint64_t gc) {
  std::memcpy(&in.m[4], &gq, 8);
  std::memcpy(&in.m[5], &gc, 8);
}

// Everything a part launch needs besides the instruction array.
struct PartLaunch {
  int64_t prog_offset;  // into the program's device instruction buffer
  int32_t nprog;
  int32_t T;            // tile bits
  int32_t RB;           // register bits
  int32_t fin_sync;     // barrier needed before the final store
  uint8_t tpos[16];     // ascending physical positions of the tile
  uint8_t fin_rpos[MAX_RB];
  uint8_t fin_npos[MAX_NPOS];
  // out-of-place launches (HS_PLAN_PINGPONG): the tile is read from buffer
  // in_buf and written to buffer out_buf (0 = state, 1 = scratch) under the
  // next layout: store slot bit r goes to physical position opos[r]
  // (ascending) and free (tile index) bit j to fpos[j]
  int32_t oop;
  int32_t in_buf, out_buf;
  int32_t cluster_log;  // tile spread over a cluster of 2^cluster_log CTAs (compiled parts only)
  uint8_t opos[16];
  uint8_t fpos[52];
  // compiled parts: the last phase's lanes 0..2 (0..3 for c64) hold store
  // slots 0..2, so registers go straight to HBM in full 128 B lines
  int32_t direct_store;
};
static_assert(sizeof(PartLaunch) == 144, "PartLaunch layout");

// A layout switch fused into an out-of-place launch (one process per GPU,
// peer memory): the launch writes every amplitude straight into the state
// buffer of the rank that owns it after the switch: segment k = the output
// index's bits at the outgoing qubits' positions pa[] -> out_ptr[k], at the
// same index with the pa bits replaced by this rank's slot (its incoming
// qubits' values).
struct FuseSwitch {
  int on = 0;
  int c = 0;                 // outgoing qubits (segment bits)
  int pa[3] = {0, 0, 0};     // their output positions, ascending
  uint64_t out_ptr[8] = {};  // per segment k: the owner's state buffer (mapped)
  int slot = 0;              // this rank's slot bits
};

struct PartPlan {
  PartLaunch launch;
  std::vector<Instr> prog;
  hs_part_info info;
  void* jit = nullptr;  // cudaKernel_t of the compiled part (HS_PLAN_JIT), else null
  double carry_in[2] = {1.0, 0.0};  // the program's pending scalar when this launch starts (jit)
  bool last = false;                // the program's last launch (applies the scalar)
  FuseSwitch fuse;
};

// Compile every plan to a straight-line kernel (hs_jit.cpp); on failure all
// plans keep jit == nullptr and the interpreter kernel runs them.
int jit_compile_program(std::vector<PartPlan>& plans, int dtype, int n_local, int device, int smem_optin,
                        std::string& err);
std::string jit_source_for(const PartPlan& pl, int dtype, int n_local);
// FP64 instructions per amplitude the compiled kernel of `pl` issues
// (the generator's count; host only, no compilation)
double jit_fp64_per_amp(const PartPlan& pl, int dtype, int n_local);
// recompile one launch of a compiled program (e.g. after setting pl.fuse)
int jit_recompile(PartPlan& pl, int dtype, int n_local, int device, int smem_optin, std::string& err);
void jit_cache_stats(int* disk_hits, int* compiles);
int jit_teams();
// on-disk cache directory ($HISVSIM_CACHE_DIR, default ~/.cache/hisvsim; empty = off)
std::string hs_cache_dir();

// Program-level qubit layout: logical position q (what parts stage) lives at
// physical bit phys[q] of the buffer. A part's write-back may permute the
// positions inside its tile (see hs_planner.cpp); inv is phys^-1.
// LAYOUT_OOP: out-of-place launch, target = the complete next layout
enum { LAYOUT_KEEP = 0, LAYOUT_PRIORITY = 1, LAYOUT_TARGET = 2, LAYOUT_OOP = 3 };
struct LayoutIO {
  const int32_t* phys_in = nullptr;   // null = identity
  const int32_t* inv_in = nullptr;
  int32_t* phys_out = nullptr;        // updated for the tile's qubits
  const int32_t* next_use = nullptr;  // PRIORITY: parts until q is staged again
  const int32_t* target = nullptr;    // TARGET: wanted physical position of q
  const int32_t* extra_first = nullptr;  // physical positions that fill the tile before the lowest free ones
  int num_extra_first = 0;
  int mode = LAYOUT_KEEP;
  int hot = 0;  // PRIORITY: lowest positions for the soonest-staged qubits (0: the default)
};

// Plan one part. Returns HS_OK or an error code with `err` filled.
int plan_part(int n_local, int dtype, int tile_max, uint32_t options, const int32_t* staged, int w,
              const hs_gate* gates, int num_gates, PartPlan& out, std::string& err,
              const LayoutIO* lay = nullptr, const int32_t* gpos = nullptr, int ng = 0);

// Plan a whole part sequence (with HS_PLAN_LAYOUT: evolving layout plus the
// restore launches that bring every qubit home at the end).
int plan_program(int n_local, int dtype, int tile_max, uint32_t options, const hs_part* parts, int num_parts,
                 const hs_gate* gates, int num_gates, std::vector<PartPlan>& plans, std::string& err,
                 std::vector<int32_t>* init_phys = nullptr, const int32_t* given_init = nullptr,
                 std::vector<int32_t>* final_phys = nullptr,
                 const std::vector<std::vector<int32_t>>* globals = nullptr);

// 2x2 base matrix of a gate kind (controls handled by masking), row-major
// complex: m[0..7] = m00 re/im, m01, m10, m11. Mirrors statevec.py:33-98.
bool base_matrix(int kind, const double* params, double m[8]);

// Structured 2x2: M = s * M' where M' has its entries snapped to 0 / +-1
// when they are within a few ulps of them. A compiled kernel evaluates each
// of the four real output components (u.re, u.im, v.re, v.im of the pair)
// as a linear combination of the inputs (x.re, x.im, y.re, y.im): a zero
// coefficient costs nothing, a +-1 coefficient turns an FMA into an add, so
// sqrt(X), sqrt(Y), H (scaled) cost 1 FP64 op per output instead of 4.
// `cost` = FP64 instructions per amplitude pair. With allow_scale, s may be
// any entry of M (the caller then owes the scalar s to every amplitude);
// without, s = 1.
struct Mat2 {
  double s[2];
  double m[8];
  int cost;
};
Mat2 structure_2x2(const double* m, bool allow_scale);
// real coefficients of output component c (0: u.re, 1: u.im, 2: v.re, 3: v.im)
// on the inputs (x.re, x.im, y.re, y.im)
void component_coefs(const double* m, int c, double coef[4]);
int component_cost(const double coef[4]);

}  // namespace hs
