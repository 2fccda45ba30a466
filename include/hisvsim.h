/*
 * hisvsim.h — C ABI of the B200-native part-pass engine (libhisvsim.so).
 *
 * The reference (HiSVSIM `hisim` 0.1.0) is pure Python/numpy and has no FFI;
 * its drop-in boundary is the Python function layer. Each
 * entry point below replaces one reference function on the hot path:
 *
 *   hs_part_apply      ~ hisim.hier.run_part          (pkg/src/hisim/hier.py:220-244)
 *                        incl. apply_op per gate      (pkg/src/hisim/statevec.py:241-261)
 *   hs_program_create  ~ hisim.hier.remap_part over all parts (hier.py:181-217),
 *                        planned once, uploaded once
 *   hs_program_run     ~ the part loop of execute_hierarchical (hier.py:342-368)
 *                        / _run_on_buffers (pkg/src/hisim/dist.py:454-482)
 *   hs_state_init_basis~ hisim.statevec.zero_state    (statevec.py:151-167)
 *   hs_bit_permute     ~ RedistributionPlan.apply, the local half
 *                        (dist.py:261-268; layout_positions dist.py:151-166)
 *   hs_pack_segments / hs_unpack_segments
 *                      ~ the remote half of RedistributionPlan.apply: gather the
 *                        amplitudes bound for each peer into contiguous
 *                        segments for the NCCL all-to-all, and scatter back
 *   hs_max_abs_diff    ~ hisim.hier.verify_against_flat (hier.py:422-436)
 *
 * Conventions (same as the reference):
 *   - amplitude index is little-endian: bit i of the index is qubit/position i;
 *   - a part is given by its staged positions (strictly ascending, the
 *     QubitSlotMap of hier.py:49-77) and its gates in program order with
 *     operands as slots into that list (ExecutablePart.op_slots), controls
 *     first and target last (qasm.py:78-88);
 *   - gate kinds are numbered in hisim.qasm.GateKind declaration order.
 *
 * Ownership: the caller owns every state buffer (device memory, e.g. a torch
 * tensor); the library never allocates or frees it. Programs and scratch are
 * owned by their handles. All launches are stream-ordered and asynchronous on
 * the stream passed in (NULL = legacy default stream). No C++ exception
 * crosses this boundary: every call returns an hs_status and the message of
 * the last failure on the calling thread is available from hs_last_error().
 */
#ifndef HISVSIM_H
#define HISVSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_ABI_VERSION 1
#define HS_MAX_STAGED 24

/* status codes; the Python shim maps them onto the hisim error taxonomy */
typedef enum {
  HS_OK = 0,
  HS_ERR_INVALID = 1,    /* ValueError: bad shape / position / operand      */
  HS_ERR_CAPACITY = 2,   /* QubitCountOutOfRangeError: does not fit          */
  HS_ERR_CUDA = 3,       /* DeviceError: CUDA runtime failure                */
  HS_ERR_TOO_WIDE = 4,   /* PartTooWideForLayoutError-like: tile > on-chip   */
  HS_ERR_UNSUPPORTED = 5 /* gate kind or dtype not supported                 */
} hs_status;

typedef enum { HS_C128 = 0, HS_C64 = 1 } hs_dtype;

/* hisim.qasm.GateKind, declaration order (qasm.py:26-47) */
typedef enum {
  HS_H = 0, HS_X, HS_Y, HS_Z, HS_S, HS_T, HS_SDG, HS_TDG,
  HS_RX, HS_RY, HS_RZ, HS_U1, HS_U3,
  HS_CX, HS_CZ, HS_CRZ, HS_CRY, HS_SWAP, HS_CCX,
  HS_NUM_KINDS
} hs_gate_kind;

/* one GateOp in slot coordinates (ExecutablePart.ops[i] + op_slots[i]) */
typedef struct {
  int32_t kind;      /* hs_gate_kind */
  int32_t num_slots; /* arity: 1, 2 or 3 */
  int32_t slots[3];  /* controls first, target last */
  int32_t reserved;
  double params[3];  /* radians, reference parameter order */
} hs_gate;

/* one part: staged positions + a window into the gate array */
typedef struct {
  int32_t num_staged;            /* w */
  int32_t staged[HS_MAX_STAGED]; /* strictly ascending, < n_local */
  int32_t gate_offset;
  int32_t num_gates;
} hs_part;

/* what the planner made of a part (for traces / reports / tests) */
typedef struct {
  int32_t tile_bits;      /* T: positions staged per CTA tile (w + fill) */
  int32_t tile_pos[32];   /* ascending physical positions of the tile */
  int32_t reg_bits;       /* register bits per thread */
  int32_t phases;         /* register phases (SMEM exchanges) */
  int32_t instructions;   /* device instructions incl. phase markers */
  int32_t dense_gates, perm_gates, diag_gates, swaps_relabelled;
  int64_t tiles;          /* CTA tiles per launch = batch * 2^(n_local - T) */
  double fp_ops_per_amp;  /* diagnostic real FLOPs per amplitude */
  int32_t input_gates;    /* gates before single-qubit fusion */
  int32_t restore;        /* 1: a layout-restore launch (no gates) */
  int32_t compiled;       /* 1: runs as an NVRTC-compiled kernel (HS_PLAN_JIT) */
  float fp64_instr_per_amp; /* FP64 pipe instructions per amplitude (FMA = 1) */
  int32_t user_part;      /* the caller's part this launch belongs to (-1: layout launch) */
} hs_part_info;

/* planner options (hs_engine_set_options / hs_plan_part) */
#define HS_PLAN_FUSE_1Q 0x1u /* merge runs of uncontrolled 1-qubit gates per qubit */
#define HS_PLAN_RB3 0x2u     /* 3 register bits per thread instead of 4 */
#define HS_PLAN_PARITY 0x4u  /* CX(a,b) D(b) CX(a,b) -> one diagonal on a xor b */
/* program-internal qubit layout: each part's write-back permutes the qubits
 * of its tile so the next parts' qubits sit in the lowest physical bits
 * (long contiguous runs); restore launches appended after the last part
 * bring the buffer back to natural order. Programs must then be run over
 * all their launches, in order. */
#define HS_PLAN_LAYOUT 0x8u
/* compile each part's program to a straight-line kernel with NVRTC (parts
 * are compiled in parallel and cached per process); if NVRTC fails the
 * interpreter kernel runs the same program */
#define HS_PLAN_JIT 0x10u
/* with HS_PLAN_LAYOUT: the program expects its initial state in a planned
 * layout (hs_program_initial_layout) instead of natural order. Meant for
 * basis-state starts, which are one amplitude in any layout. */
#define HS_PLAN_INIT_LAYOUT 0x20u
/* with HS_PLAN_LAYOUT: parts run out of place, alternating between the state
 * and a scratch buffer of the same size (hs_program_bind_scratch), so each
 * part can write any layout: the next part's qubits on the lowest bits, and
 * the last part natural order (no restore launches). An odd part count runs
 * part 0 in place. */
#define HS_PLAN_PINGPONG 0x40u
/* parts wider than one CTA's tile (k = 13, 14 complex128): run each as one
 * compiled cluster-tile pass (needs HS_PLAN_JIT). Without it such a part runs
 * as a short sequence of passes over sub-parts of its gates that fit the tile
 * (the hierarchical idea one level down; same results). */
#define HS_PLAN_CLUSTER 0x80u
/* with HS_PLAN_LAYOUT: leave the buffer in the program's final layout
 * (hs_program_final_layout) instead of restoring natural order, e.g. when a
 * layout switch that can pack from any layout follows */
#define HS_PLAN_NO_RESTORE 0x100u
/* wide parts (HS_PLAN_CLUSTER off): split each part on its own instead of
 * regrouping the whole program's gate stream into tile-sized passes (the
 * default when that takes fewer passes; a pass may then carry the end of
 * one part and the start of the next) */
#define HS_PLAN_PART_LOCAL 0x200u
/* regroup the gate stream into tile-sized passes even when every part fits
 * the tile (fewer launches than parts when consecutive parts together fit
 * one tile; same results, launches report the part they mostly carry) */
#define HS_PLAN_MERGE 0x400u
/* with HS_PLAN_MERGE | HS_PLAN_JIT | HS_PLAN_PARITY: diagonal gates (Z-type
 * 1-qubit gates, CZ, CRZ, CX.D.CX parity diagonals) need not have their
 * qubits staged - a compiled pass applies them from the tile's free index
 * bits - so regrouped passes stage only the qubits their non-diagonal gates
 * act on (fewer passes; kept when the grouping takes fewer launches) */
#define HS_PLAN_GLOBAL_DIAG 0x800u
#define HS_PLAN_DEFAULT (HS_PLAN_FUSE_1Q | HS_PLAN_PARITY | HS_PLAN_MERGE | HS_PLAN_GLOBAL_DIAG)

typedef struct hs_engine hs_engine;
typedef struct hs_program hs_program;

const char* hs_last_error(void);
int hs_abi_version(void);

/* engine: binds a CUDA device; holds launch configuration */
int hs_engine_create(int device, hs_engine** out);
int hs_engine_destroy(hs_engine* eng);
/* SMs and the max tile bits per dtype chosen for this device */
int hs_engine_query(hs_engine* eng, int* num_sms, int* tile_bits_c128, int* tile_bits_c64);
/* planner options for programs created afterwards (HS_PLAN_* bits) */
int hs_engine_set_options(hs_engine* eng, uint32_t options);

/* plan + upload a whole part sequence for buffers of batch x 2^n_local */
int hs_program_create(hs_engine* eng, int n_local, int dtype,
                      const hs_part* parts, int num_parts,
                      const hs_gate* gates, int num_gates, hs_program** out);
/* the same for a buffer that arrives in a given layout: logical position q
 * at physical bit init_phys[q] (a permutation; needs HS_PLAN_LAYOUT set on
 * the engine). The program still ends in natural order. Used after an
 * in-place layout switch (hs_pack/unpack_segments_range). */
int hs_program_create_from_layout(hs_engine* eng, int n_local, int dtype,
                                  const hs_part* parts, int num_parts,
                                  const hs_gate* gates, int num_gates,
                                  const int32_t* init_phys, hs_program** out);
int hs_program_destroy(hs_program* prog);
int hs_program_num_parts(hs_program* prog);
/* launches = parts + layout-restore launches (HS_PLAN_LAYOUT) */
int hs_program_num_launches(hs_program* prog);
/* per launch (index < num_launches) */
int hs_program_part_info(hs_program* prog, int part, hs_part_info* out);
/* physical bit of each logical position in the state the program expects
 * (phys[n_local]; identity unless HS_PLAN_INIT_LAYOUT). Basis state |x>
 * lives at index sum_q bit_q(x) << phys[q]. */
int hs_program_initial_layout(hs_program* prog, int32_t* phys);
/* physical bit of each logical position after the program's last launch
 * (identity unless HS_PLAN_NO_RESTORE) */
int hs_program_final_layout(hs_program* prog, int32_t* phys);
/* scratch buffer for HS_PLAN_PINGPONG programs: device memory of at least
 * the state's size, owned by the caller, used by every later run */
int hs_program_bind_scratch(hs_program* prog, void* scratch, size_t bytes);
/* empty unless HS_PLAN_JIT compilation failed (the interpreter then runs) */
const char* hs_program_jit_error(hs_program* prog);
/* Fuse a layout switch into launch `launch` of a compiled ping-pong program
 * (one process per GPU, peer memory): instead of writing its tile to this
 * rank's state, the launch writes it to the state buffer of the rank that
 * owns it after the switch - out_ptrs[k] (a device pointer, e.g. an IPC
 * mapping of that rank's state) for the amplitudes whose output index's bits
 * at the outgoing qubits' positions seg_pos[] (ascending) spell k - at the
 * same index with those bits replaced by my_slot. This is the
 * in-place switch of hs_group_switch without the pack and pull passes: the
 * transfer rides on the pass's stores. The launch must be out of place and
 * write the state (out_buf 0); every rank's previous launch must be complete
 * before any rank runs it (it overwrites peers' state buffers). num_seg_bits
 * = 0 with out_ptrs NULL restores the plain launch. Recompiles the launch. */
int hs_program_fuse_switch(hs_program* prog, int launch, int num_seg_bits, const int32_t* seg_pos,
                           const uint64_t* out_ptrs, int32_t my_slot);
/* process-wide counts of compiled-part kernels loaded from the on-disk cubin
 * cache ($HISVSIM_CACHE_DIR, default ~/.cache/hisvsim; "off" disables) and
 * compiled with NVRTC (in-process cache hits count as neither) */
int hs_jit_cache_stats(int* disk_hits, int* compiles);
/* device instructions of one launch, copied to host (test/debug); returns the
 * count via *count; buf may be NULL to query the size in bytes */
int hs_program_dump(hs_program* prog, int part, void* buf, size_t buf_bytes,
                    int* count, size_t* instr_bytes);
/* launch [first, first+count) of the program's launches in order on
 * `stream` over `batch` contiguous rows of 2^n_local amplitudes each */
int hs_program_run(hs_program* prog, void* state, int64_t batch,
                   int first, int count, void* stream);
/* same, but records the launches into a CUDA graph on first use and
 * replays it afterwards (state pointer and batch must not change) */
int hs_program_run_graph(hs_program* prog, void* state, int64_t batch, void* stream);

/* host-only planning of one part (no CUDA call; usable without a GPU):
 * writes the PartLaunch header + device instructions into buf (NULL to
 * query *bytes), and the plan summary into *info */
int hs_plan_part(int n_local, int dtype, int tile_bits, uint32_t options, const int32_t* staged, int w,
                 const hs_gate* gates, int num_gates, void* buf, size_t buf_bytes,
                 size_t* bytes, hs_part_info* info);

/* host-only planning of a whole program (layout + restore launches
 * included): buf receives, per launch, a PartLaunch header followed by its
 * instructions (NULL to query *bytes); *num_launches is set */
int hs_plan_program(int n_local, int dtype, int tile_bits, uint32_t options,
                    const hs_part* parts, int num_parts, const hs_gate* gates, int num_gates,
                    void* buf, size_t buf_bytes, size_t* bytes, int* num_launches);

/* host-only: the layouts a program would run with (what
 * hs_program_initial_layout / hs_program_final_layout report for the same
 * plan) and its launch count; either array may be NULL */
int hs_plan_program_layouts(int n_local, int dtype, int tile_bits, uint32_t options, const hs_part* parts,
                            int num_parts, const hs_gate* gates, int num_gates, int32_t* init_phys,
                            int32_t* final_phys, int* num_launches);

/* CUDA C++ source of the compiled (HS_PLAN_JIT) kernel of one part, as
 * generated from its plan (host-only; tests compile it with nvcc) */
int hs_jit_source(int n_local, int dtype, int tile_bits, uint32_t options, const int32_t* staged, int w,
                  const hs_gate* gates, int num_gates, char* buf, size_t buf_bytes, size_t* bytes);

/* dagP merge phase (hisim partition.py:396-478, partition_dagp's greedy pair
 * contraction) on the host: groups with qubit masks and group-level DAG
 * edges in, the surviving group of every group out; identical merges to
 * the reference. Host-only; circuits of at most 64 qubits. */
int hs_dagp_merge(int num_groups, const uint64_t* qmask, int num_edges, const int32_t* edge_src,
                  const int32_t* edge_dst, int limit, int32_t* merged_into);

/* the structured form compiled kernels use for a 2x2 gate matrix m
 * (row-major complex, 8 doubles): m = s * m_out with m_out's entries
 * snapped to 0 / +-1 within a few ulps; returns the FP64 instructions per
 * amplitude pair (allow_scale = 0: s = 1). Host-only. */
int hs_structure_2x2(const double* m, int allow_scale, double* s_out, double* m_out);

/* one-shot run_part: plan, upload, launch, free (synchronizes the stream) */
int hs_part_apply(hs_engine* eng, void* state, int64_t batch, int n_local, int dtype,
                  const int32_t* staged, int w, const hs_gate* gates, int num_gates,
                  void* stream);

/* |index> : zero the buffer and write 1 at `index` (per row when batch>1 use
 * row 0 only: the buffer is treated as one state of batch*2^n_local) */
int hs_state_init_basis(void* state, int64_t num_amps, int dtype, int64_t index, void* stream);

/* out[perm(i)] = in[i] where bit j of i moves to bit dst_of[j];
 * out-of-place, num_bits <= 40 */
int hs_bit_permute(const void* in, void* out, int num_bits, int dtype,
                   const int32_t* dst_of, void* stream);

/* measured FP64 FMA throughput of the current device (a DFMA-chain
 * microbenchmark, ~20 ms): the denominator of the FP64 roofline */
int hs_fp64_peak(double* tflops, void* stream);

/* max |a - b| over n amplitudes of `dtype`, b given as complex128 (the
 * oracle's type); result written to *host_result after a stream sync */
int hs_max_abs_diff(const void* a, int dtype, const void* b_c128, int64_t n,
                    double* host_result, void* stream);

/* Pack for a qubit-remap all-to-all: with `num_seg_bits` local positions
 * seg_pos[] whose values name a destination segment, copy src into dst so
 * that all amplitudes of segment k are contiguous (segment-major, inner
 * order = remaining bits ascending). unpack is the inverse. */
int hs_pack_segments(const void* src, void* dst, int num_bits, int dtype,
                     const int32_t* seg_pos, int num_seg_bits, void* stream);
int hs_unpack_segments(const void* src, void* dst, int num_bits, int dtype,
                       const int32_t* seg_pos, int num_seg_bits, void* stream);

/* Ranged forms for in-place chunked switches: only inner offsets
 * [inner_begin, inner_begin + inner_count) of every segment move; packed
 * index = k * inner_count + (m - inner_begin). */
int hs_pack_segments_range(const void* src, void* dst, int num_bits, int dtype,
                           const int32_t* seg_pos, int num_seg_bits,
                           int64_t inner_begin, int64_t inner_count, void* stream);
int hs_unpack_segments_range(const void* src, void* dst, int num_bits, int dtype,
                             const int32_t* seg_pos, int num_seg_bits,
                             int64_t inner_begin, int64_t inner_count, void* stream);

/* Pull form of the unpack (a layout switch over peer memory): packed
 * element m of slot k is read from src_by_slot[k][m] - a device pointer that
 * may live on another GPU (peer access or an IPC mapping) - and written to
 * inner offset inner_begin + m of segment k of dst. 2^num_seg_bits pointers. */
int hs_unpack_segments_range_from(const void* const* src_by_slot, void* dst, int num_bits, int dtype,
                                  const int32_t* seg_pos, int num_seg_bits, int64_t inner_begin,
                                  int64_t inner_count, void* stream);

/* Multi-device engine: 2^p shards driven by one process, shard r on
 * devices[r] (several shards may share a device; distinct devices get peer
 * access over NVLink / NVSwitch). Two staging buffers of staging_bytes per
 * shard. Replaces the exchange of RedistributionPlan.apply
 * (pkg/src/hisim/dist.py:261-268) across GPUs. */
typedef struct hs_group hs_group;
int hs_group_create(int num_shards, const int32_t* devices, size_t staging_bytes, hs_group** out);
int hs_group_destroy(hs_group* group);
/* In-place qubit-remap switch of every shard (2^n_local amplitudes each):
 * the num_seg_bits positions seg_pos[] (ascending) of shard r spell a
 * segment k that moves to shard seg_dst[r << num_seg_bits | k], where it
 * lands in the positions of its segment src_slot[r]; the other bits keep
 * their positions. Chunk by chunk of inner offsets: every shard packs its
 * outgoing segments into local staging, then pulls its incoming segments
 * from the senders' staging over peer memory into its own shard. Launches
 * on streams[r] (a NULL entry is the legacy default stream; a NULL array:
 * the group's own streams) with cross-shard event ordering; asynchronous
 * unless *seconds is requested (then the max over shards of the switch's
 * device time is written after a sync). */
int hs_group_switch(hs_group* group, void* const* shards, int n_local, int dtype, const int32_t* seg_pos,
                    int num_seg_bits, const int32_t* seg_dst, const int32_t* src_slot, void* const* streams,
                    double* seconds);
/* one process per GPU: export / map another process's device buffer
 * (cudaIpcMemHandle_t, 64 bytes) so hs_unpack_segments_range_from can pull
 * from a peer's staging. Buffers to export come from hs_device_alloc (a
 * whole allocation: the mapped pointer is its base). */
int hs_device_alloc(size_t bytes, void** device_ptr);
/* let kernels on the current device read / write peer_device's memory
 * (NVLink / NVSwitch); a no-op for the current device itself */
int hs_enable_peer_access(int peer_device);
int hs_device_free(void* device_ptr);
int hs_ipc_get_handle(const void* device_ptr, void* handle_out);
int hs_ipc_open_handle(const void* handle, void** device_ptr);
int hs_ipc_close(void* device_ptr);

#ifdef __cplusplus
}
#endif
#endif /* HISVSIM_H */
