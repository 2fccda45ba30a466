// C-ABI implementation (include/hisvsim.h): engine and program handles,
// status codes + thread-local last error, stream-ordered launches.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "hs_common.h"

namespace hs {
cudaError_t prepare_kernels(int smem_optin);
cudaError_t launch_part(int dtype, const PartLaunch& L, const Instr* dprog, void* psi, void* psi_out, int n_local,
                        int64_t batch, int num_sms, cudaStream_t stream);
cudaError_t launch_set_basis(void* psi, int dtype, int64_t index, cudaStream_t s);
cudaError_t launch_bit_permute(const void* in, void* out, int nbits, int dtype, const int32_t* dst_of,
                               int num_sms, cudaStream_t s);
cudaError_t launch_segments_range(bool pack, const void* in, void* out, int nbits, int dtype, const int32_t* seg_pos,
                                  int nseg, int64_t begin, int64_t count, int num_sms, cudaStream_t s);
cudaError_t launch_segments(bool pack, const void* in, void* out, int nbits, int dtype,
                            const int32_t* seg_pos, int nseg, int num_sms, cudaStream_t s);
cudaError_t launch_maxdiff(const void* a, int dtype, const void* b, int64_t n, unsigned long long* dres,
                           int num_sms, cudaStream_t s);
cudaError_t measure_fp64_peak(double* tflops, int num_sms, cudaStream_t s);
cudaError_t launch_segments_from(const void* const* src, void* out, int nbits, int dtype, const int32_t* seg_pos,
                                 int nseg, int64_t begin, int64_t count, int num_sms, cudaStream_t s);
}  // namespace hs

using namespace hs;

struct hs_engine {
  int device = 0;
  int num_sms = 0;
  int smem_optin = 0;
  int tile_c128 = 12;
  int tile_c64 = 13;
  uint32_t options = HS_PLAN_DEFAULT;
  unsigned long long* d_scratch = nullptr;  // reductions
};

// A group of 2^p shards driven by one process: each shard on its own device
// (peer access enabled between distinct devices) or several on one device.
// Layout switches move amplitudes between shards over peer memory
// (NVLink / NVSwitch), in place and chunk by chunk: pack the chunk's
// outgoing segments into local staging, then every shard pulls its incoming
// segments straight from the owners' staging into its own positions.
struct hs_group {
  int num_shards = 0;
  std::vector<int> devices;
  std::vector<int> sms;
  size_t staging_bytes = 0;           // per staging buffer (two per shard)
  std::vector<void*> staging[2];      // [buffer][shard]
  std::vector<cudaStream_t> streams;  // one per shard (non-blocking)
  std::vector<cudaEvent_t> packed[2], pulled[2], t0, t1;
};

struct hs_program {
  hs_engine* eng = nullptr;
  int n_local = 0;
  int dtype = 0;
  int user_parts = 0;            // plans beyond this are layout-restore launches
  std::vector<int32_t> init_phys; // layout the program expects its input in
  std::vector<int32_t> final_phys; // layout the program leaves the buffer in
  void* scratch = nullptr;        // HS_PLAN_PINGPONG partner buffer (caller-owned)
  size_t scratch_bytes = 0;
  std::string jit_error;         // why HS_PLAN_JIT fell back to the interpreter
  std::vector<PartPlan> plans;
  Instr* d_prog = nullptr;
  cudaGraphExec_t graph = nullptr;
  void* graph_state = nullptr;
  void* graph_scratch = nullptr;
  int64_t graph_batch = 0;
  cudaStream_t graph_stream = nullptr;
  int teams = 2;  // teams per CTA of the compiled kernels (jit_teams at compile time)
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(HS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                               cudaGetErrorString(e) + ")");
}

#define HS_CUDA(call, what)                         \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

int tile_for(const hs_engine* eng, int dtype) {
  return dtype == HS_C128 ? eng->tile_c128 : eng->tile_c64;
}

int check_dtype(int dtype) {
  if (dtype != HS_C128 && dtype != HS_C64) return fail(HS_ERR_UNSUPPORTED, "dtype must be HS_C128 or HS_C64");
  return HS_OK;
}

}  // namespace

extern "C" {

const char* hs_last_error(void) { return g_err.c_str(); }
int hs_abi_version(void) { return HS_ABI_VERSION; }

int hs_engine_create(int device, hs_engine** out) {
  if (!out) return fail(HS_ERR_INVALID, "out is NULL");
  *out = nullptr;
  int count = 0;
  HS_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  if (device < 0 || device >= count)
    return fail(HS_ERR_INVALID, "device " + std::to_string(device) + " outside 0.." + std::to_string(count - 1));
  HS_CUDA(cudaSetDevice(device), "cudaSetDevice");
  int major = 0;
  HS_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device), "attr");
  if (major != 10) return fail(HS_ERR_UNSUPPORTED, "libhisvsim is built for sm_100a (B200) only");
  std::unique_ptr<hs_engine> eng(new (std::nothrow) hs_engine);
  if (!eng) return fail(HS_ERR_CAPACITY, "out of host memory");
  eng->device = device;
  HS_CUDA(cudaDeviceGetAttribute(&eng->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
  HS_CUDA(cudaDeviceGetAttribute(&eng->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "attr");
  HS_CUDA(prepare_kernels(eng->smem_optin), "cudaFuncSetAttribute");
  HS_CUDA(cudaMalloc(&eng->d_scratch, 64), "cudaMalloc scratch");
  *out = eng.release();
  return HS_OK;
}

int hs_engine_destroy(hs_engine* eng) {
  if (!eng) return HS_OK;
  cudaSetDevice(eng->device);
  if (eng->d_scratch) cudaFree(eng->d_scratch);
  delete eng;
  return HS_OK;
}

int hs_engine_query(hs_engine* eng, int* num_sms, int* tile_c128, int* tile_c64) {
  if (!eng) return fail(HS_ERR_INVALID, "engine is NULL");
  if (num_sms) *num_sms = eng->num_sms;
  if (tile_c128) *tile_c128 = eng->tile_c128;
  if (tile_c64) *tile_c64 = eng->tile_c64;
  return HS_OK;
}

static int program_create(hs_engine* eng, int n_local, int dtype, const hs_part* parts, int num_parts,
                          const hs_gate* gates, int num_gates, const int32_t* init_phys, hs_program** out);

int hs_program_create(hs_engine* eng, int n_local, int dtype, const hs_part* parts, int num_parts,
                      const hs_gate* gates, int num_gates, hs_program** out) {
  return program_create(eng, n_local, dtype, parts, num_parts, gates, num_gates, nullptr, out);
}

int hs_program_create_from_layout(hs_engine* eng, int n_local, int dtype, const hs_part* parts, int num_parts,
                                  const hs_gate* gates, int num_gates, const int32_t* init_phys, hs_program** out) {
  if (!init_phys) return fail(HS_ERR_INVALID, "init_phys is NULL");
  if (!eng || !(eng->options & HS_PLAN_LAYOUT)) return fail(HS_ERR_INVALID, "a given initial layout needs HS_PLAN_LAYOUT");
  if (n_local < 1 || n_local > 62) return fail(HS_ERR_INVALID, "n_local outside [1, 62]");
  std::vector<char> seen(n_local, 0);
  for (int q = 0; q < n_local; ++q) {
    if (init_phys[q] < 0 || init_phys[q] >= n_local || seen[init_phys[q]])
      return fail(HS_ERR_INVALID, "init_phys is not a permutation of 0..n_local-1");
    seen[init_phys[q]] = 1;
  }
  return program_create(eng, n_local, dtype, parts, num_parts, gates, num_gates, init_phys, out);
}

static int program_create(hs_engine* eng, int n_local, int dtype, const hs_part* parts, int num_parts,
                          const hs_gate* gates, int num_gates, const int32_t* init_phys, hs_program** out) {
  if (!eng || !out) return fail(HS_ERR_INVALID, "engine/out is NULL");
  *out = nullptr;
  if (int s = check_dtype(dtype)) return s;
  if (num_parts < 0 || (num_parts > 0 && !parts)) return fail(HS_ERR_INVALID, "bad part array");
  std::unique_ptr<hs_program> prog(new (std::nothrow) hs_program);
  if (!prog) return fail(HS_ERR_CAPACITY, "out of host memory");
  prog->eng = eng;
  prog->n_local = n_local;
  prog->dtype = dtype;
  {
    std::string err;
    // compiled parts: 256-thread teams (2^(T - 4)) keep 128 registers per
    // thread, so complex64 tiles are 12 bits there too
    const int tile = (eng->options & HS_PLAN_JIT) ? std::min(tile_for(eng, dtype), 12) : tile_for(eng, dtype);
    int s = plan_program(n_local, dtype, tile, eng->options, parts, num_parts, gates, num_gates,
                         prog->plans, err, &prog->init_phys, init_phys, &prog->final_phys);
    if (s != HS_OK) return fail(s, err);
  }
  prog->user_parts = num_parts;
  if (eng->options & HS_PLAN_JIT) {
    std::string err;
    prog->teams = jit_teams();
    HS_CUDA(cudaSetDevice(eng->device), "cudaSetDevice");
    int s = jit_compile_program(prog->plans, dtype, n_local, eng->device, eng->smem_optin, err);
    if (s != HS_OK) prog->jit_error = err;  // interpreter fallback on the GPU, reported
  }
  // passes with global (unstaged) diagonal qubits exist only as compiled
  // kernels: the interpreter cannot run them
  for (const auto& pl : prog->plans)
    if (!pl.jit && !pl.prog.empty() && pl.prog[0].op == I_GLOBALS)
      return fail(HS_ERR_UNSUPPORTED, "compiled passes failed (" + prog->jit_error +
                                           "); passes with global diagonal qubits have no interpreter form");
  size_t total = 0;
  for (auto& pl : prog->plans) {
    pl.launch.prog_offset = (int64_t)total;
    total += pl.prog.size();
  }
  if (total) {
    HS_CUDA(cudaSetDevice(eng->device), "cudaSetDevice");
    std::vector<Instr> all;
    all.reserve(total);
    for (auto& pl : prog->plans) all.insert(all.end(), pl.prog.begin(), pl.prog.end());
    HS_CUDA(cudaMalloc(&prog->d_prog, total * sizeof(Instr)), "cudaMalloc program");
    HS_CUDA(cudaMemcpy(prog->d_prog, all.data(), total * sizeof(Instr), cudaMemcpyHostToDevice),
            "cudaMemcpy program");
  }
  *out = prog.release();
  return HS_OK;
}

int hs_program_destroy(hs_program* prog) {
  if (!prog) return HS_OK;
  cudaSetDevice(prog->eng->device);
  if (prog->graph) cudaGraphExecDestroy(prog->graph);
  if (prog->d_prog) cudaFree(prog->d_prog);
  delete prog;
  return HS_OK;
}

int hs_program_num_parts(hs_program* prog) { return prog ? prog->user_parts : -1; }

int hs_program_num_launches(hs_program* prog) { return prog ? (int)prog->plans.size() : -1; }

int hs_program_part_info(hs_program* prog, int part, hs_part_info* out) {
  if (!prog || !out) return fail(HS_ERR_INVALID, "program/out is NULL");
  if (part < 0 || part >= (int)prog->plans.size()) return fail(HS_ERR_INVALID, "part index out of range");
  *out = prog->plans[part].info;
  out->compiled = prog->plans[part].jit != nullptr;
  return HS_OK;
}

int hs_program_dump(hs_program* prog, int part, void* buf, size_t buf_bytes, int* count,
                    size_t* instr_bytes) {
  if (!prog) return fail(HS_ERR_INVALID, "program is NULL");
  if (part < 0 || part >= (int)prog->plans.size()) return fail(HS_ERR_INVALID, "part index out of range");
  const PartPlan& pl = prog->plans[part];
  if (count) *count = (int)pl.prog.size();
  if (instr_bytes) *instr_bytes = sizeof(Instr);
  // layout: PartLaunch header followed by the instructions
  const size_t need = sizeof(PartLaunch) + pl.prog.size() * sizeof(Instr);
  if (!buf) return HS_OK;
  if (buf_bytes < need) return fail(HS_ERR_INVALID, "dump buffer too small");
  std::memcpy(buf, &pl.launch, sizeof(PartLaunch));
  std::memcpy((char*)buf + sizeof(PartLaunch), pl.prog.data(), pl.prog.size() * sizeof(Instr));
  return HS_OK;
}

static int run_range(hs_program* prog, void* state, int64_t batch, int first, int count, cudaStream_t s) {
  hs_engine* eng = prog->eng;
  const size_t need = size_t(batch) << prog->n_local;
  for (int i = first; i < first + count; ++i) {
    const PartPlan& pl = prog->plans[i];
    if ((pl.launch.in_buf || pl.launch.out_buf) &&
        (!prog->scratch || prog->scratch_bytes < need * (prog->dtype == HS_C128 ? 16 : 8)))
      return fail(HS_ERR_INVALID, "ping-pong program: bind a scratch buffer of the state's size first");
    void* bufs[2] = {state, prog->scratch};
    void* psi = bufs[pl.launch.in_buf];
    void* psi_out = bufs[pl.launch.out_buf];
    if (pl.jit && pl.launch.cluster_log > 0) {
      // cluster tile: clusters of 2^cluster_log CTAs (one per SM), each CTA
      // two teams over three buffers of 2^(T - cluster_log) slots (hs_jit.cpp)
      long long ntiles = (long long)(batch << (prog->n_local - pl.launch.T));
      void* args[] = {&psi, &psi_out, &ntiles};
      const int csize = 1 << pl.launch.cluster_log;
      const int TC = pl.launch.T - pl.launch.cluster_log;
      long long nclusters = (long long)eng->num_sms / csize;
      if (nclusters > (ntiles + 1) / 2) nclusters = (ntiles + 1) / 2;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(nclusters * csize));
      cfg.blockDim = dim3(2u << (TC - pl.launch.RB));
      cfg.dynamicSmemBytes = 3 * (size_t(prog->dtype == HS_C128 ? 16 : 8) << TC) + 128;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = csize;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      HS_CUDA(cudaLaunchKernelExC(&cfg, (const void*)pl.jit, args), "compiled cluster-tile part launch");
      continue;
    }
    if (pl.jit) {
      long long ntiles = (long long)(batch << (prog->n_local - pl.launch.T));
      void* args[] = {&psi, &psi_out, &ntiles};
      // one CTA per SM, two teams, three tile buffers + their mbarriers (hs_jit.cpp)
      const size_t smem = 3 * (size_t(prog->dtype == HS_C128 ? 16 : 8) << pl.launch.T) + 64;
      long long grid = (long long)eng->num_sms;
      const int teams = prog->teams;
      if (grid > (ntiles + teams - 1) / teams) grid = (ntiles + teams - 1) / teams;
      HS_CUDA(cudaLaunchKernel((const void*)pl.jit, dim3((unsigned)grid),
                               dim3((unsigned)teams << (pl.launch.T - pl.launch.RB)), args, smem, s),
              "compiled part kernel launch");
      continue;
    }
    HS_CUDA(launch_part(prog->dtype, pl.launch, prog->d_prog, psi, psi_out, prog->n_local, batch, eng->num_sms, s),
            "part kernel launch");
  }
  return HS_OK;
}

int hs_program_bind_scratch(hs_program* prog, void* scratch, size_t bytes) {
  if (!prog) return fail(HS_ERR_INVALID, "program is NULL");
  prog->scratch = scratch;
  prog->scratch_bytes = scratch ? bytes : 0;
  return HS_OK;
}

int hs_program_final_layout(hs_program* prog, int32_t* phys) {
  if (!prog || !phys) return fail(HS_ERR_INVALID, "program/phys is NULL");
  for (int q = 0; q < prog->n_local; ++q)
    phys[q] = q < (int)prog->final_phys.size() ? prog->final_phys[q] : q;
  return HS_OK;
}

int hs_program_initial_layout(hs_program* prog, int32_t* phys) {
  if (!prog || !phys) return fail(HS_ERR_INVALID, "program/phys is NULL");
  for (int q = 0; q < prog->n_local; ++q)
    phys[q] = q < (int)prog->init_phys.size() ? prog->init_phys[q] : q;
  return HS_OK;
}

const char* hs_program_jit_error(hs_program* prog) { return prog ? prog->jit_error.c_str() : ""; }

int hs_program_fuse_switch(hs_program* prog, int launch, int num_seg_bits, const int32_t* seg_pos,
                           const uint64_t* out_ptrs, int32_t my_slot) {
  if (!prog) return fail(HS_ERR_INVALID, "program is NULL");
  if (launch < 0 || launch >= (int)prog->plans.size()) return fail(HS_ERR_INVALID, "launch index out of range");
  PartPlan& pl = prog->plans[launch];
  if (num_seg_bits == 0 && !out_ptrs) {  // clear
    if (!pl.fuse.on) return HS_OK;
    pl.fuse = FuseSwitch();
  } else {
    if (!pl.jit) return fail(HS_ERR_UNSUPPORTED, "a fused switch needs a compiled launch (HS_PLAN_JIT)");
    if (!pl.launch.oop || pl.launch.out_buf != 0 || pl.launch.cluster_log)
      return fail(HS_ERR_UNSUPPORTED, "a fused switch needs an out-of-place launch that writes the state");
    if (num_seg_bits < 1 || num_seg_bits > 3 || !seg_pos || !out_ptrs)
      return fail(HS_ERR_INVALID, "a fused switch moves 1..3 qubits");
    FuseSwitch f;
    f.on = 1;
    f.c = num_seg_bits;
    for (int b = 0; b < num_seg_bits; ++b) {
      f.pa[b] = seg_pos[b];
      if (seg_pos[b] < 0 || seg_pos[b] >= prog->n_local || (b && seg_pos[b] <= seg_pos[b - 1]))
        return fail(HS_ERR_INVALID, "segment positions must be ascending positions of the shard");
    }
    for (int k = 0; k < (1 << num_seg_bits); ++k) {
      if (!out_ptrs[k]) return fail(HS_ERR_INVALID, "NULL destination");
      f.out_ptr[k] = out_ptrs[k];
    }
    if (my_slot < 0 || my_slot >= (1 << num_seg_bits)) return fail(HS_ERR_INVALID, "slot outside the segments");
    f.slot = my_slot;
    pl.fuse = f;
  }
  std::string err;
  HS_CUDA(cudaSetDevice(prog->eng->device), "cudaSetDevice");
  if (int s = jit_recompile(pl, prog->dtype, prog->n_local, prog->eng->device, prog->eng->smem_optin, err))
    return fail(s, err);
  if (prog->graph) {  // the captured graph holds the old kernel
    cudaGraphExecDestroy(prog->graph);
    prog->graph = nullptr;
  }
  return HS_OK;
}

int hs_jit_cache_stats(int* disk_hits, int* compiles) {
  jit_cache_stats(disk_hits, compiles);
  return HS_OK;
}

int hs_program_run(hs_program* prog, void* state, int64_t batch, int first, int count, void* stream) {
  if (!prog || !state) return fail(HS_ERR_INVALID, "program/state is NULL");
  if (batch < 1) return fail(HS_ERR_INVALID, "batch must be >= 1");
  if (first < 0 || count < 0 || first + count > (int)prog->plans.size())
    return fail(HS_ERR_INVALID, "part range outside the program");
  HS_CUDA(cudaSetDevice(prog->eng->device), "cudaSetDevice");
  return run_range(prog, state, batch, first, count, (cudaStream_t)stream);
}

int hs_program_run_graph(hs_program* prog, void* state, int64_t batch, void* stream) {
  if (!prog || !state) return fail(HS_ERR_INVALID, "program/state is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  HS_CUDA(cudaSetDevice(prog->eng->device), "cudaSetDevice");
  if (prog->graph && (prog->graph_state != state || prog->graph_batch != batch || prog->graph_scratch != prog->scratch)) {
    cudaGraphExecDestroy(prog->graph);
    prog->graph = nullptr;
  }
  if (!prog->graph) {
    cudaStream_t cap = s;
    bool own = false;
    if (!cap) {  // cannot capture the legacy stream
      HS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "cudaStreamCreate");
      own = true;
    }
    HS_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
    int st = run_range(prog, state, batch, 0, (int)prog->plans.size(), cap);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cap, &g);
    if (st != HS_OK) { if (g) cudaGraphDestroy(g); if (own) cudaStreamDestroy(cap); return st; }
    if (e != cudaSuccess) { if (own) cudaStreamDestroy(cap); return cuda_fail(e, "end capture"); }
    e = cudaGraphInstantiate(&prog->graph, g, 0);
    cudaGraphDestroy(g);
    if (own) cudaStreamDestroy(cap);
    if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
    prog->graph_state = state;
    prog->graph_batch = batch;
    prog->graph_scratch = prog->scratch;
  }
  HS_CUDA(cudaGraphLaunch(prog->graph, s), "graph launch");
  return HS_OK;
}

int hs_engine_set_options(hs_engine* eng, uint32_t options) {
  if (!eng) return fail(HS_ERR_INVALID, "engine is NULL");
  eng->options = options;
  return HS_OK;
}

int hs_plan_part(int n_local, int dtype, int tile_bits, uint32_t options, const int32_t* staged, int w,
                 const hs_gate* gates, int num_gates, void* buf, size_t buf_bytes, size_t* bytes,
                 hs_part_info* info) {
  if (int s = check_dtype(dtype)) return s;
  if (num_gates < 0 || (num_gates > 0 && !gates) || (w > 0 && !staged)) return fail(HS_ERR_INVALID, "bad arrays");
  if (tile_bits < 1 || tile_bits > MAX_TILE) return fail(HS_ERR_INVALID, "tile_bits outside [1, 13]");
  PartPlan plan;
  std::string err;
  int s = plan_part(n_local, dtype, tile_bits, options, staged, w, gates, num_gates, plan, err);
  if (s != HS_OK) return fail(s, err);
  const size_t need = sizeof(PartLaunch) + plan.prog.size() * sizeof(Instr);
  if (bytes) *bytes = need;
  if (info) *info = plan.info;
  if (!buf) return HS_OK;
  if (buf_bytes < need) return fail(HS_ERR_INVALID, "plan buffer too small");
  plan.launch.prog_offset = 0;
  std::memcpy(buf, &plan.launch, sizeof(PartLaunch));
  std::memcpy((char*)buf + sizeof(PartLaunch), plan.prog.data(), plan.prog.size() * sizeof(Instr));
  return HS_OK;
}

int hs_plan_program(int n_local, int dtype, int tile_bits, uint32_t options, const hs_part* parts, int num_parts,
                    const hs_gate* gates, int num_gates, void* buf, size_t buf_bytes, size_t* bytes,
                    int* num_launches) {
  if (int s = check_dtype(dtype)) return s;
  if (num_parts < 0 || (num_parts > 0 && !parts)) return fail(HS_ERR_INVALID, "bad part array");
  if (tile_bits < 1 || tile_bits > MAX_TILE) return fail(HS_ERR_INVALID, "tile_bits outside [1, 13]");
  std::vector<PartPlan> plans;
  std::string err;
  int s = plan_program(n_local, dtype, tile_bits, options, parts, num_parts, gates, num_gates, plans, err);
  if (s != HS_OK) return fail(s, err);
  size_t need = 0;
  for (auto& pl : plans) need += sizeof(PartLaunch) + pl.prog.size() * sizeof(Instr);
  if (bytes) *bytes = need;
  if (num_launches) *num_launches = (int)plans.size();
  if (const char* dir = std::getenv("HISVSIM_DUMP_SRC")) {
    // debugging aid: the generated source of every compiled launch
    for (size_t i = 0; i < plans.size(); ++i) {
      if (!(options & HS_PLAN_JIT)) break;
      std::string path = std::string(dir) + "/launch" + std::to_string(i) + ".cu";
      if (FILE* f = std::fopen(path.c_str(), "w")) {
        std::string src = jit_source_for(plans[i], dtype, n_local);
        std::fwrite(src.data(), 1, src.size(), f);
        std::fclose(f);
      }
    }
  }
  if (!buf) return HS_OK;
  if (buf_bytes < need) return fail(HS_ERR_INVALID, "plan buffer too small");
  char* o = (char*)buf;
  for (auto& pl : plans) {
    pl.launch.prog_offset = 0;
    std::memcpy(o, &pl.launch, sizeof(PartLaunch));
    o += sizeof(PartLaunch);
    std::memcpy(o, pl.prog.data(), pl.prog.size() * sizeof(Instr));
    o += pl.prog.size() * sizeof(Instr);
  }
  return HS_OK;
}

int hs_plan_program_layouts(int n_local, int dtype, int tile_bits, uint32_t options, const hs_part* parts,
                            int num_parts, const hs_gate* gates, int num_gates, int32_t* init_phys,
                            int32_t* final_phys, int* num_launches) {
  if (int s = check_dtype(dtype)) return s;
  if (num_parts < 0 || (num_parts > 0 && !parts)) return fail(HS_ERR_INVALID, "bad part array");
  if (tile_bits < 1 || tile_bits > MAX_TILE) return fail(HS_ERR_INVALID, "tile_bits outside [1, 13]");
  std::vector<PartPlan> plans;
  std::vector<int32_t> ip, fp;
  std::string err;
  int s = plan_program(n_local, dtype, tile_bits, options, parts, num_parts, gates, num_gates, plans, err, &ip,
                       nullptr, &fp);
  if (s != HS_OK) return fail(s, err);
  for (int q = 0; q < n_local; ++q) {
    if (init_phys) init_phys[q] = q < (int)ip.size() ? ip[q] : q;
    if (final_phys) final_phys[q] = q < (int)fp.size() ? fp[q] : q;
  }
  if (num_launches) *num_launches = (int)plans.size();
  return HS_OK;
}

int hs_jit_source(int n_local, int dtype, int tile_bits, uint32_t options, const int32_t* staged, int w,
                  const hs_gate* gates, int num_gates, char* buf, size_t buf_bytes, size_t* bytes) {
  if (int s = check_dtype(dtype)) return s;
  if (tile_bits < 1 || tile_bits > MAX_TILE) return fail(HS_ERR_INVALID, "tile_bits outside [1, 13]");
  PartPlan plan;
  std::string err;
  int s = plan_part(n_local, dtype, tile_bits, options, staged, w, gates, num_gates, plan, err);
  if (s != HS_OK) return fail(s, err);
  std::string src = jit_source_for(plan, dtype, n_local);
  if (bytes) *bytes = src.size() + 1;
  if (!buf) return HS_OK;
  if (buf_bytes < src.size() + 1) return fail(HS_ERR_INVALID, "source buffer too small");
  std::memcpy(buf, src.c_str(), src.size() + 1);
  return HS_OK;
}

int hs_structure_2x2(const double* m, int allow_scale, double* s_out, double* m_out) {
  if (!m) return -1;
  Mat2 r = structure_2x2(m, allow_scale != 0);
  if (s_out) { s_out[0] = r.s[0]; s_out[1] = r.s[1]; }
  if (m_out) std::memcpy(m_out, r.m, sizeof(r.m));
  return r.cost;
}

int hs_part_apply(hs_engine* eng, void* state, int64_t batch, int n_local, int dtype, const int32_t* staged,
                  int w, const hs_gate* gates, int num_gates, void* stream) {
  if (!eng || !state) return fail(HS_ERR_INVALID, "engine/state is NULL");
  hs_part part;
  std::memset(&part, 0, sizeof(part));
  if (w < 0 || w > HS_MAX_STAGED) return fail(HS_ERR_INVALID, "staged count outside [0, 24]");
  part.num_staged = w;
  for (int j = 0; j < w; ++j) part.staged[j] = staged[j];
  part.gate_offset = 0;
  part.num_gates = num_gates;
  // a one-shot part never plans an initial layout of its own: the caller's
  // buffer is in natural order and must be left in natural order
  const uint32_t saved = eng->options;
  eng->options &= ~(uint32_t)(HS_PLAN_INIT_LAYOUT | HS_PLAN_NO_RESTORE);
  hs_program* prog = nullptr;
  int s = hs_program_create(eng, n_local, dtype, &part, 1, gates, num_gates, &prog);
  eng->options = saved;
  if (s != HS_OK) return s;
  void* scratch = nullptr;
  bool pingpong = false;
  for (const PartPlan& pl : prog->plans) pingpong |= pl.launch.in_buf || pl.launch.out_buf;
  cudaStream_t cs = (cudaStream_t)stream;
  if (pingpong) {  // out-of-place launches: a scratch copy for the program's lifetime
    const size_t bytes = (size_t(batch) << n_local) * (dtype == HS_C128 ? 16 : 8);
    cudaError_t e = cudaMallocAsync(&scratch, bytes, cs);
    if (e != cudaSuccess) { hs_program_destroy(prog); return cuda_fail(e, "cudaMallocAsync scratch"); }
    hs_program_bind_scratch(prog, scratch, bytes);
  }
  // every launch of the plan: a part can take several (tile-sized
  // sub-passes of a wide part, layout restores, the deferred scalar)
  s = hs_program_run(prog, state, batch, 0, (int)prog->plans.size(), stream);
  if (scratch) cudaFreeAsync(scratch, cs);
  if (s == HS_OK) {
    cudaError_t e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) s = cuda_fail(e, "stream sync");
  }
  hs_program_destroy(prog);
  return s;
}

int hs_state_init_basis(void* state, int64_t num_amps, int dtype, int64_t index, void* stream) {
  if (!state) return fail(HS_ERR_INVALID, "state is NULL");
  if (int s = check_dtype(dtype)) return s;
  if (index < 0 || index >= num_amps) return fail(HS_ERR_INVALID, "basis index outside the state");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t amp = dtype == HS_C128 ? 16 : 8;
  HS_CUDA(cudaMemsetAsync(state, 0, amp * (size_t)num_amps, s), "cudaMemsetAsync");
  HS_CUDA(launch_set_basis(state, dtype, index, s), "set basis");
  return HS_OK;
}

static int sms_of_current() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

int hs_bit_permute(const void* in, void* out, int num_bits, int dtype, const int32_t* dst_of, void* stream) {
  if (!in || !out || !dst_of) return fail(HS_ERR_INVALID, "NULL argument");
  if (in == out) return fail(HS_ERR_INVALID, "hs_bit_permute is out-of-place");
  if (int s = check_dtype(dtype)) return s;
  if (num_bits < 0 || num_bits > 40) return fail(HS_ERR_INVALID, "num_bits outside [0, 40]");
  uint64_t seen = 0;
  for (int b = 0; b < num_bits; ++b) {
    if (dst_of[b] < 0 || dst_of[b] >= num_bits || (seen >> dst_of[b] & 1))
      return fail(HS_ERR_INVALID, "dst_of is not a permutation");
    seen |= 1ull << dst_of[b];
  }
  HS_CUDA(launch_bit_permute(in, out, num_bits, dtype, dst_of, sms_of_current(), (cudaStream_t)stream),
          "bit permute");
  return HS_OK;
}

static int segments(bool pack, const void* src, void* dst, int num_bits, int dtype, const int32_t* seg_pos,
                    int nseg, void* stream) {
  if (!src || !dst || (nseg && !seg_pos)) return fail(HS_ERR_INVALID, "NULL argument");
  if (src == dst) return fail(HS_ERR_INVALID, "pack/unpack are out-of-place");
  if (int s = check_dtype(dtype)) return s;
  if (nseg < 0 || nseg > 8 || num_bits < nseg || num_bits > 40)
    return fail(HS_ERR_INVALID, "segment bits outside range");
  for (int k = 0; k < nseg; ++k) {
    if (seg_pos[k] < 0 || seg_pos[k] >= num_bits) return fail(HS_ERR_INVALID, "segment position outside state");
    if (k && seg_pos[k] <= seg_pos[k - 1]) return fail(HS_ERR_INVALID, "segment positions not ascending");
  }
  HS_CUDA(launch_segments(pack, src, dst, num_bits, dtype, seg_pos, nseg, sms_of_current(), (cudaStream_t)stream),
          "segment kernel");
  return HS_OK;
}

int hs_pack_segments(const void* src, void* dst, int num_bits, int dtype, const int32_t* seg_pos, int nseg,
                     void* stream) {
  return segments(true, src, dst, num_bits, dtype, seg_pos, nseg, stream);
}

int hs_unpack_segments(const void* src, void* dst, int num_bits, int dtype, const int32_t* seg_pos, int nseg,
                       void* stream) {
  return segments(false, src, dst, num_bits, dtype, seg_pos, nseg, stream);
}

static int segments_range(bool pack, const void* src, void* dst, int num_bits, int dtype, const int32_t* seg_pos,
                          int nseg, int64_t inner_begin, int64_t inner_count, void* stream) {
  if (!src || !dst || (nseg && !seg_pos)) return fail(HS_ERR_INVALID, "NULL argument");
  if (src == dst) return fail(HS_ERR_INVALID, "pack/unpack are out-of-place");
  if (int s = check_dtype(dtype)) return s;
  if (nseg < 0 || nseg > 8 || num_bits < nseg || num_bits > 62)
    return fail(HS_ERR_INVALID, "segment bits outside range");
  for (int k = 0; k < nseg; ++k) {
    if (seg_pos[k] < 0 || seg_pos[k] >= num_bits) return fail(HS_ERR_INVALID, "segment position outside state");
    if (k && seg_pos[k] <= seg_pos[k - 1]) return fail(HS_ERR_INVALID, "segment positions not ascending");
  }
  const int64_t inner = int64_t(1) << (num_bits - nseg);
  if (inner_begin < 0 || inner_count < 0 || inner_begin + inner_count > inner)
    return fail(HS_ERR_INVALID, "inner range outside the segments");
  if (inner_count == 0) return HS_OK;
  HS_CUDA(launch_segments_range(pack, src, dst, num_bits, dtype, seg_pos, nseg, inner_begin, inner_count,
                                sms_of_current(), (cudaStream_t)stream),
          "segment range kernel");
  return HS_OK;
}

int hs_pack_segments_range(const void* src, void* dst, int num_bits, int dtype, const int32_t* seg_pos, int nseg,
                           int64_t inner_begin, int64_t inner_count, void* stream) {
  return segments_range(true, src, dst, num_bits, dtype, seg_pos, nseg, inner_begin, inner_count, stream);
}

int hs_unpack_segments_range(const void* src, void* dst, int num_bits, int dtype, const int32_t* seg_pos, int nseg,
                             int64_t inner_begin, int64_t inner_count, void* stream) {
  return segments_range(false, src, dst, num_bits, dtype, seg_pos, nseg, inner_begin, inner_count, stream);
}

int hs_unpack_segments_range_from(const void* const* src_by_slot, void* dst, int num_bits, int dtype,
                                  const int32_t* seg_pos, int nseg, int64_t inner_begin, int64_t inner_count,
                                  void* stream) {
  if (!src_by_slot || !dst || (nseg && !seg_pos)) return fail(HS_ERR_INVALID, "NULL argument");
  if (int s = check_dtype(dtype)) return s;
  if (nseg < 0 || nseg > 8 || num_bits < nseg || num_bits > 62)
    return fail(HS_ERR_INVALID, "segment bits outside range");
  for (int k = 0; k < nseg; ++k) {
    if (seg_pos[k] < 0 || seg_pos[k] >= num_bits) return fail(HS_ERR_INVALID, "segment position outside state");
    if (k && seg_pos[k] <= seg_pos[k - 1]) return fail(HS_ERR_INVALID, "segment positions not ascending");
  }
  for (int k = 0; k < (1 << nseg); ++k)
    if (!src_by_slot[k]) return fail(HS_ERR_INVALID, "NULL source slot");
  const int64_t inner = int64_t(1) << (num_bits - nseg);
  if (inner_begin < 0 || inner_count < 0 || inner_begin + inner_count > inner)
    return fail(HS_ERR_INVALID, "inner range outside the segments");
  if (inner_count == 0) return HS_OK;
  HS_CUDA(launch_segments_from(src_by_slot, dst, num_bits, dtype, seg_pos, nseg, inner_begin, inner_count,
                               sms_of_current(), (cudaStream_t)stream),
          "segment pull kernel");
  return HS_OK;
}

int hs_group_create(int num_shards, const int32_t* devices, size_t staging_bytes, hs_group** out) {
  if (!out || !devices) return fail(HS_ERR_INVALID, "NULL argument");
  *out = nullptr;
  if (num_shards < 1 || num_shards > 256 || (num_shards & (num_shards - 1)))
    return fail(HS_ERR_INVALID, "num_shards must be a power of two in [1, 256]");
  if (staging_bytes < 4096) return fail(HS_ERR_INVALID, "staging_bytes below 4 KiB");
  int count = 0;
  HS_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  for (int r = 0; r < num_shards; ++r)
    if (devices[r] < 0 || devices[r] >= count) return fail(HS_ERR_INVALID, "device index outside the node");
  std::unique_ptr<hs_group> g(new (std::nothrow) hs_group);
  if (!g) return fail(HS_ERR_CAPACITY, "out of host memory");
  g->num_shards = num_shards;
  g->devices.assign(devices, devices + num_shards);
  g->staging_bytes = staging_bytes;
  // peer access between every pair of distinct devices (NVLink / NVSwitch)
  for (int a : g->devices)
    for (int b : g->devices) {
      if (a == b) continue;
      int ok = 0;
      HS_CUDA(cudaDeviceCanAccessPeer(&ok, a, b), "cudaDeviceCanAccessPeer");
      if (!ok) return fail(HS_ERR_UNSUPPORTED, "devices " + std::to_string(a) + " and " + std::to_string(b) +
                                                     " have no peer access");
      HS_CUDA(cudaSetDevice(a), "cudaSetDevice");
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    }
  auto cleanup = [](hs_group* h) { hs_group_destroy(h); };
  std::unique_ptr<hs_group, decltype(cleanup)> guard(g.release(), cleanup);
  hs_group* G = guard.get();
  for (int b = 0; b < 2; ++b) {
    G->staging[b].assign(num_shards, nullptr);
    G->packed[b].assign(num_shards, nullptr);
    G->pulled[b].assign(num_shards, nullptr);
  }
  G->streams.assign(num_shards, nullptr);
  G->t0.assign(num_shards, nullptr);
  G->t1.assign(num_shards, nullptr);
  G->sms.assign(num_shards, 0);
  for (int r = 0; r < num_shards; ++r) {
    HS_CUDA(cudaSetDevice(G->devices[r]), "cudaSetDevice");
    HS_CUDA(cudaDeviceGetAttribute(&G->sms[r], cudaDevAttrMultiProcessorCount, G->devices[r]), "attr");
    HS_CUDA(cudaStreamCreateWithFlags(&G->streams[r], cudaStreamNonBlocking), "cudaStreamCreate");
    for (int b = 0; b < 2; ++b) {
      HS_CUDA(cudaMalloc(&G->staging[b][r], staging_bytes), "cudaMalloc staging");
      HS_CUDA(cudaEventCreateWithFlags(&G->packed[b][r], cudaEventDisableTiming), "cudaEventCreate");
      HS_CUDA(cudaEventCreateWithFlags(&G->pulled[b][r], cudaEventDisableTiming), "cudaEventCreate");
    }
    HS_CUDA(cudaEventCreate(&G->t0[r]), "cudaEventCreate");
    HS_CUDA(cudaEventCreate(&G->t1[r]), "cudaEventCreate");
  }
  *out = guard.release();
  return HS_OK;
}

int hs_group_destroy(hs_group* g) {
  if (!g) return HS_OK;
  for (int r = 0; r < g->num_shards; ++r) {
    if (r < (int)g->devices.size()) cudaSetDevice(g->devices[r]);
    for (int b = 0; b < 2; ++b) {
      if (r < (int)g->staging[b].size() && g->staging[b][r]) cudaFree(g->staging[b][r]);
      if (r < (int)g->packed[b].size() && g->packed[b][r]) cudaEventDestroy(g->packed[b][r]);
      if (r < (int)g->pulled[b].size() && g->pulled[b][r]) cudaEventDestroy(g->pulled[b][r]);
    }
    if (r < (int)g->t0.size() && g->t0[r]) cudaEventDestroy(g->t0[r]);
    if (r < (int)g->t1.size() && g->t1[r]) cudaEventDestroy(g->t1[r]);
    if (r < (int)g->streams.size() && g->streams[r]) cudaStreamDestroy(g->streams[r]);
  }
  delete g;
  return HS_OK;
}

int hs_group_switch(hs_group* g, void* const* shards, int n_local, int dtype, const int32_t* seg_pos, int nseg,
                    const int32_t* seg_dst, const int32_t* src_slot, void* const* streams, double* seconds) {
  if (!g || !shards || !seg_dst || !src_slot || (nseg && !seg_pos)) return fail(HS_ERR_INVALID, "NULL argument");
  if (int s = check_dtype(dtype)) return s;
  if (nseg < 0 || nseg > 8 || n_local < nseg || n_local > 62) return fail(HS_ERR_INVALID, "segment bits outside range");
  const int R = g->num_shards, S = 1 << nseg;
  for (int k = 0; k < nseg; ++k)
    if (seg_pos[k] < 0 || seg_pos[k] >= n_local || (k && seg_pos[k] <= seg_pos[k - 1]))
      return fail(HS_ERR_INVALID, "segment positions must be ascending positions of the shard");
  // who pulls what: slot j of shard r comes from the source s whose data
  // lands in slot j (src_slot[s] == j) and whose segment k goes to r
  std::vector<int32_t> from_src((size_t)R * S, -1), from_seg((size_t)R * S, -1);
  for (int s = 0; s < R; ++s) {
    if (src_slot[s] < 0 || src_slot[s] >= S) return fail(HS_ERR_INVALID, "src_slot outside the segments");
    for (int k = 0; k < S; ++k) {
      const int d = seg_dst[(size_t)s * S + k];
      if (d < 0 || d >= R) return fail(HS_ERR_INVALID, "seg_dst outside the group");
      int32_t& f = from_src[(size_t)d * S + src_slot[s]];
      if (f >= 0) return fail(HS_ERR_INVALID, "two segments land in the same slot of a shard");
      f = s;
      from_seg[(size_t)d * S + src_slot[s]] = k;
    }
  }
  for (size_t i = 0; i < from_src.size(); ++i)
    if (from_src[i] < 0) return fail(HS_ERR_INVALID, "a slot of a shard receives nothing");
  const size_t amp = dtype == HS_C128 ? 16 : 8;
  const int64_t inner = int64_t(1) << (n_local - nseg);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(inner, int64_t(g->staging_bytes / (amp * S))));
  // a given array is taken as is (a NULL entry is the legacy default stream)
  auto stream_of = [&](int r) { return streams ? (cudaStream_t)streams[r] : g->streams[r]; };
  if (seconds)
    for (int r = 0; r < R; ++r) {
      HS_CUDA(cudaSetDevice(g->devices[r]), "cudaSetDevice");
      HS_CUDA(cudaEventRecord(g->t0[r], stream_of(r)), "cudaEventRecord");
    }
  std::vector<const void*> srcs(S);
  int m = 0;
  for (int64_t begin = 0; begin < inner; begin += chunk, ++m) {
    const int64_t cnt = std::min(chunk, inner - begin);
    const int b = m & 1;
    for (int r = 0; r < R; ++r) {
      HS_CUDA(cudaSetDevice(g->devices[r]), "cudaSetDevice");
      cudaStream_t st = stream_of(r);
      // staging buffer b was last read by the pulls of chunk m - 2
      if (m >= 2)
        for (int s = 0; s < R; ++s) HS_CUDA(cudaStreamWaitEvent(st, g->pulled[b][s], 0), "wait");
      HS_CUDA(launch_segments_range(true, shards[r], g->staging[b][r], n_local, dtype, seg_pos, nseg, begin, cnt,
                                    g->sms[r], st),
              "pack");
      HS_CUDA(cudaEventRecord(g->packed[b][r], st), "cudaEventRecord");
    }
    for (int r = 0; r < R; ++r) {
      HS_CUDA(cudaSetDevice(g->devices[r]), "cudaSetDevice");
      cudaStream_t st = stream_of(r);
      for (int j = 0; j < S; ++j) {
        const int s = from_src[(size_t)r * S + j];
        HS_CUDA(cudaStreamWaitEvent(st, g->packed[b][s], 0), "wait");
        srcs[j] = (const char*)g->staging[b][s] + (size_t)from_seg[(size_t)r * S + j] * cnt * amp;
      }
      HS_CUDA(launch_segments_from(srcs.data(), shards[r], n_local, dtype, seg_pos, nseg, begin, cnt, g->sms[r], st),
              "pull");
      HS_CUDA(cudaEventRecord(g->pulled[b][r], st), "cudaEventRecord");
    }
  }
  // no shard runs ahead into the next pass before every pull has read its data
  for (int r = 0; r < R; ++r) {
    HS_CUDA(cudaSetDevice(g->devices[r]), "cudaSetDevice");
    for (int s = 0; s < R; ++s)
      for (int b = 0; b < 2 && b < m; ++b) HS_CUDA(cudaStreamWaitEvent(stream_of(r), g->pulled[b][s], 0), "wait");
  }
  if (seconds) {
    double worst = 0;
    for (int r = 0; r < R; ++r) {
      HS_CUDA(cudaSetDevice(g->devices[r]), "cudaSetDevice");
      HS_CUDA(cudaEventRecord(g->t1[r], stream_of(r)), "cudaEventRecord");
    }
    for (int r = 0; r < R; ++r) {
      HS_CUDA(cudaEventSynchronize(g->t1[r]), "cudaEventSynchronize");
      float ms = 0;
      HS_CUDA(cudaEventElapsedTime(&ms, g->t0[r], g->t1[r]), "cudaEventElapsedTime");
      worst = std::max(worst, double(ms) / 1e3);
    }
    *seconds = worst;
  }
  return HS_OK;
}

int hs_enable_peer_access(int peer_device) {
  int dev = 0, ok = 0;
  HS_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  if (peer_device == dev) return HS_OK;
  HS_CUDA(cudaDeviceCanAccessPeer(&ok, dev, peer_device), "cudaDeviceCanAccessPeer");
  if (!ok) return fail(HS_ERR_UNSUPPORTED, "device " + std::to_string(dev) + " has no peer access to device " +
                                               std::to_string(peer_device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
  else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return HS_OK;
}

int hs_device_alloc(size_t bytes, void** device_ptr) {
  if (!device_ptr) return fail(HS_ERR_INVALID, "NULL argument");
  *device_ptr = nullptr;
  if (bytes == 0) return fail(HS_ERR_INVALID, "zero-byte allocation");
  cudaError_t e = cudaMalloc(device_ptr, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(HS_ERR_CAPACITY, "cudaMalloc of " + std::to_string(bytes) + " bytes: out of device memory");
  }
  HS_CUDA(e, "cudaMalloc");
  return HS_OK;
}

int hs_device_free(void* device_ptr) {
  if (device_ptr) HS_CUDA(cudaFree(device_ptr), "cudaFree");
  return HS_OK;
}

int hs_ipc_get_handle(const void* device_ptr, void* handle_out) {
  if (!device_ptr || !handle_out) return fail(HS_ERR_INVALID, "NULL argument");
  cudaIpcMemHandle_t h;
  HS_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(device_ptr)), "cudaIpcGetMemHandle");
  std::memcpy(handle_out, &h, sizeof(h));
  return HS_OK;
}

int hs_ipc_open_handle(const void* handle, void** device_ptr) {
  if (!handle || !device_ptr) return fail(HS_ERR_INVALID, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  HS_CUDA(cudaIpcOpenMemHandle(device_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return HS_OK;
}

int hs_ipc_close(void* device_ptr) {
  if (!device_ptr) return fail(HS_ERR_INVALID, "NULL argument");
  HS_CUDA(cudaIpcCloseMemHandle(device_ptr), "cudaIpcCloseMemHandle");
  return HS_OK;
}

int hs_fp64_peak(double* tflops, void* stream) {
  if (!tflops) return fail(HS_ERR_INVALID, "NULL argument");
  HS_CUDA(measure_fp64_peak(tflops, sms_of_current(), (cudaStream_t)stream), "fp64 probe");
  return HS_OK;
}

int hs_max_abs_diff(const void* a, int dtype, const void* b_c128, int64_t n, double* host_result, void* stream) {
  if (!a || !b_c128 || !host_result) return fail(HS_ERR_INVALID, "NULL argument");
  if (int s = check_dtype(dtype)) return s;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* d = nullptr;
  HS_CUDA(cudaMallocAsync((void**)&d, sizeof(unsigned long long), s), "cudaMallocAsync");
  HS_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s), "memset");
  if (n > 0) HS_CUDA(launch_maxdiff(a, dtype, b_c128, n, d, sms_of_current(), s), "maxdiff");
  unsigned long long bits = 0;
  HS_CUDA(cudaMemcpyAsync(&bits, d, sizeof(bits), cudaMemcpyDeviceToHost, s), "memcpy");
  HS_CUDA(cudaFreeAsync(d, s), "cudaFreeAsync");
  HS_CUDA(cudaStreamSynchronize(s), "sync");
  double r;
  std::memcpy(&r, &bits, sizeof(r));
  *host_result = r;
  return HS_OK;
}

}  // extern "C"
