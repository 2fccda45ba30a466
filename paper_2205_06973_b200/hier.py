"""Partitioned execution on the B200: one kernel pass per part.

API mirror of ``hisim.hier`` (/root/reference/pkg/src/hisim/hier.py).
The reference gathers, for every fixing of the qubits outside a part, the
2^w amplitudes the part touches, applies the part's gates and scatters them
back (``run_part``, hier.py:220-244), batched over all fixings in numpy.
Here the same pass is one launch of the part kernel (csrc/hs_kernels.cu):
each CTA stages one fixing-tile in shared memory and registers, applies all
of the part's gates on chip and writes back once, so a part costs one HBM
read and one HBM write of the state.

Host-side addressing helpers (``QubitSlotMap``, ``bit_offsets``,
``part_block_indices``, ``gather``, ``scatter``) and the executable-part
descriptor (``remap_part``) keep the reference's exact semantics; the slot
map and op slots are what the C ABI consumes.
"""

from __future__ import annotations

import ctypes
import json
from bisect import bisect_left
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Sequence

import numpy as np

from . import _native
from .errors import VerificationError
from .partition import MultiLevelPartition, Part, PartitionResult
from .qasm import Circuit, GateKind, GateOp
from .statevec import StateVector, allocate, default_device, from_numpy, init_basis, native_dtype, zero_state

__all__ = [
    "QubitSlotMap", "ExecutablePart", "PartTrace", "ExecutionTrace", "PartProgram",
    "bit_offsets", "part_block_indices", "gather", "scatter", "remap_part", "run_part",
    "execute_hierarchical", "execute_multilevel", "verify_against_flat",
]

_KIND_CODE = {k: i for i, k in enumerate(GateKind)}

#: programs over states of at least this many local qubits compile their
#: parts to straight-line kernels (HS_PLAN_JIT) unless options say otherwise
JIT_MIN_QUBITS = 20
#: ... and plan the coalescing layout (HS_PLAN_LAYOUT) from this size on
LAYOUT_MIN_QUBITS = 23
#: free HBM left over after the ping-pong scratch buffer is allocated
PINGPONG_HEADROOM = 2 << 30


# --- addressing (host) --------------------------------------------------------

@dataclass(frozen=True)
class QubitSlotMap:
    """Outer bit positions (strictly ascending); slot i <-> qubits[i]."""

    qubits: tuple[int, ...]

    def __post_init__(self) -> None:
        q = self.qubits
        if any(b <= a for a, b in zip(q, q[1:])):
            raise ValueError(f"positions not strictly ascending: {q}")
        if q and q[0] < 0:
            raise ValueError(f"negative position: {q[0]}")

    @property
    def num_slots(self) -> int:
        return len(self.qubits)

    def slot_of(self, q: int) -> int:
        i = bisect_left(self.qubits, q)
        if i == len(self.qubits) or self.qubits[i] != q:
            raise KeyError(f"position {q} not in slot map {self.qubits}")
        return i

    def global_of(self, slot: int) -> int:
        return self.qubits[slot]


def bit_offsets(bits: Sequence[int]) -> np.ndarray:
    """Entry k = sum of 2^bits[j] over the set bits j of k (hier.py:80-91)."""
    k = np.arange(1 << len(bits), dtype=np.int64)
    out = np.zeros_like(k)
    for j, b in enumerate(bits):
        out |= ((k >> j) & 1) << b
    return out


def _validate_positions(num_qubits: int, qubits: Sequence[int]) -> list[int]:
    if len(set(qubits)) != len(qubits):
        raise ValueError(f"duplicate positions in {qubits}")
    for q in qubits:
        if not 0 <= q < num_qubits:
            raise ValueError(f"position {q} outside 0..{num_qubits - 1}")
    inside = set(qubits)
    return [q for q in range(num_qubits) if q not in inside]


def part_block_indices(num_qubits: int, qubits: Sequence[int]) -> np.ndarray:
    """(2^f, 2^w) index matrix: row a = fixing a of the free bits (ascending),
    column s = inner index over ``qubits`` (hier.py:94-109)."""
    free = _validate_positions(num_qubits, qubits)
    return bit_offsets(free)[:, None] + bit_offsets(list(qubits))[None, :]


def _row(num_qubits: int, qubits: Sequence[int], free_index: int) -> np.ndarray:
    free = _validate_positions(num_qubits, qubits)
    if not 0 <= free_index < (1 << len(free)):
        raise ValueError(f"free_index {free_index} outside 0..{(1 << len(free)) - 1}")
    base = 0
    for j, b in enumerate(free):
        base |= ((free_index >> j) & 1) << b
    return np.int64(base) + bit_offsets(list(qubits))


def gather(data, num_qubits: int, qubits: Sequence[int], free_index: int):
    """Copy one inner vector (one fixing of the free bits) out of ``data``."""
    idx = _row(num_qubits, qubits, free_index)
    if isinstance(data, np.ndarray):
        return data[idx].copy()
    import torch

    return data[torch.as_tensor(idx, device=data.device)].clone()


def scatter(data, num_qubits: int, qubits: Sequence[int], free_index: int, inner) -> None:
    """Write an inner vector back where ``gather`` read it."""
    idx = _row(num_qubits, qubits, free_index)
    if tuple(inner.shape) != idx.shape:
        raise ValueError(f"inner has shape {tuple(inner.shape)}, need {idx.shape}")
    if isinstance(data, np.ndarray):
        data[idx] = inner
        return
    import torch

    data[torch.as_tensor(idx, device=data.device)] = inner


# --- executable parts -------------------------------------------------------------

@dataclass(frozen=True)
class ExecutablePart:
    """A part in inner-vector coordinates (hier.py:159-178): ``slot_map``
    holds the outer positions, ``op_slots`` the gate operands as slots."""

    part_id: int
    gate_indices: tuple[int, ...]
    slot_map: QubitSlotMap
    ops: tuple[GateOp, ...]
    op_slots: tuple[tuple[int, ...], ...]

    @property
    def num_slots(self) -> int:
        return self.slot_map.num_slots


def remap_part(
    circuit: Circuit,
    part: Part,
    *,
    position_of: Mapping[int, int] | None = None,
    stage_qubits: Iterable[int] | None = None,
) -> ExecutablePart:
    """Executable form of ``part`` (hier.py:181-217): ``position_of``
    re-addresses global qubits (rank-local offsets, level-1 slots);
    ``stage_qubits`` widens the staged set (must cover the part)."""
    if stage_qubits is None:
        staged = part.qubits
    else:
        staged = tuple(sorted(stage_qubits))
        if not set(part.qubits) <= set(staged):
            raise ValueError(f"stage set {staged} does not cover part qubits {part.qubits}")
    if position_of is None:
        positions = tuple(staged)
    else:
        positions = tuple(sorted(position_of[q] for q in staged))
        if len(set(positions)) != len(staged):
            raise ValueError("position_of maps two staged qubits to one position")
    smap = QubitSlotMap(positions)
    where = (lambda q: q) if position_of is None else (lambda q: position_of[q])
    ops = tuple(circuit.ops[g] for g in part.gate_indices)
    op_slots = tuple(tuple(smap.slot_of(where(q)) for q in op.qubits) for op in ops)
    return ExecutablePart(part.id, part.gate_indices, smap, ops, op_slots)


def _pack(exes: Sequence[ExecutablePart]):
    """ExecutableParts -> (hs_part[], hs_gate[]) for the C ABI."""
    total = sum(len(e.ops) for e in exes)
    parts = (_native.HsPart * max(1, len(exes)))()
    gates = (_native.HsGate * max(1, total))()
    g = 0
    for i, e in enumerate(exes):
        if e.num_slots > _native.HS_MAX_STAGED:
            raise ValueError(f"part {e.part_id} stages {e.num_slots} > {_native.HS_MAX_STAGED} positions")
        p = parts[i]
        p.num_staged = e.num_slots
        for j, q in enumerate(e.slot_map.qubits):
            p.staged[j] = q
        p.gate_offset = g
        p.num_gates = len(e.ops)
        for op, slots in zip(e.ops, e.op_slots):
            rec = gates[g]
            rec.kind = _KIND_CODE[op.kind]
            rec.num_slots = len(slots)
            for a, s in enumerate(slots):
                rec.slots[a] = s
            for a, v in enumerate(op.params):
                rec.params[a] = float(v)
            g += 1
    return parts, gates, total


class PartProgram:
    """A planned, device-resident sequence of parts for buffers of
    ``rows x 2^n_local`` amplitudes (hs_program_create). Planning happens
    once; ``run`` only launches."""

    def __init__(self, n_local: int, exes: Sequence[ExecutablePart], dtype="complex128", device=None,
                 options: int | None = None, basis_start: bool = False, init_layout: Sequence[int] | None = None,
                 final_natural: bool = True):
        """``options``: planner bits (``_native.HS_PLAN_*``); default: the
        engine default plus ``HS_PLAN_JIT`` / ``HS_PLAN_LAYOUT`` by state
        size. ``basis_start``: the program will only be run on basis states
        prepared with :meth:`init_basis`, so it may pick its initial layout
        (``HS_PLAN_INIT_LAYOUT``; ``run`` then expects that layout).
        ``init_layout``: the buffer arrives with logical position q on
        physical bit ``init_layout[q]`` (after an in-place layout switch);
        the program ends in natural order unless ``final_natural`` is False
        (then the buffer stays in ``final_layout``; a layout switch packs
        from it)."""
        import torch

        self.n_local = n_local
        self.dtype = torch.complex64 if str(dtype) in ("complex64", "c64", "torch.complex64") else torch.complex128
        self.device = torch.device(device) if device is not None else default_device()
        self.num_parts = len(exes)
        lib = _native.load()
        dev = self.device.index if self.device.index is not None else 0
        eng = _native.engine(dev)
        if options is None:
            options = _native.default_options()
            widest = max((e.num_slots for e in exes), default=0)
            if n_local >= JIT_MIN_QUBITS or widest > (12 if self.dtype == torch.complex128 else 13):
                # (parts wider than one CTA's tile only run as compiled cluster tiles)
                # compiling a part costs ~0.5-1 s of host time (parallel over
                # parts, cached); worth it once a pass moves >= 32 MiB
                options |= _native.HS_PLAN_JIT
            if n_local >= LAYOUT_MIN_QUBITS:
                # coalescing layout + restore launches pay off once the state
                # streams from HBM (measured: c2/c3 win, the L2-resident c1 loses)
                options |= _native.HS_PLAN_LAYOUT
                if basis_start:
                    options |= _native.HS_PLAN_INIT_LAYOUT
                # out-of-place parts (any next layout, no restore launches)
                # when a scratch copy of the state fits next to it (counted
                # as if the state were not allocated yet)
                amp = 16 if self.dtype == torch.complex128 else 8
                from .statevec import free_bytes

                free = free_bytes(self.device)
                if 2 * (amp << n_local) + PINGPONG_HEADROOM <= free:
                    options |= _native.HS_PLAN_PINGPONG
        if init_layout is not None and tuple(init_layout) != tuple(range(n_local)):
            options |= _native.HS_PLAN_LAYOUT
            options &= ~_native.HS_PLAN_INIT_LAYOUT
        else:
            init_layout = None
        if not final_natural and options & _native.HS_PLAN_LAYOUT:
            options |= _native.HS_PLAN_NO_RESTORE
        self.options = options
        parts, gates, total = _pack(exes)
        out = ctypes.c_void_p()
        code = 0 if self.dtype == torch.complex128 else 1
        with torch.cuda.device(self.device):
            _native.check(lib.hs_engine_set_options(eng, options))
            try:
                if init_layout is None:
                    _native.check(lib.hs_program_create(eng, n_local, code, parts, len(exes), gates, total,
                                                        ctypes.byref(out)))
                else:
                    phys = (ctypes.c_int32 * n_local)(*[int(x) for x in init_layout])
                    _native.check(lib.hs_program_create_from_layout(eng, n_local, code, parts, len(exes), gates,
                                                                    total, phys, ctypes.byref(out)))
            finally:
                lib.hs_engine_set_options(eng, _native.default_options())
        self._h = out.value
        self._lib = lib
        self.num_launches = lib.hs_program_num_launches(self._h)
        self.jit_error = lib.hs_program_jit_error(self._h).decode(errors="replace")
        self._scratch = None
        phys = (ctypes.c_int32 * max(1, n_local))()
        _native.check(lib.hs_program_initial_layout(self._h, phys))
        #: physical bit of each qubit in the state ``run`` expects
        self.initial_layout = tuple(int(phys[q]) for q in range(n_local))
        _native.check(lib.hs_program_final_layout(self._h, phys))
        #: ... and the layout ``run`` leaves it in (natural unless final_natural=False)
        self.final_layout = tuple(int(phys[q]) for q in range(n_local))

    def basis_index(self, index: int) -> int:
        """Where basis state |index> lives in the program's initial layout."""
        return sum(((index >> q) & 1) << p for q, p in enumerate(self.initial_layout))

    def init_basis(self, data, index: int = 0) -> None:
        """Prepare |index> in the layout ``run`` expects."""
        from .statevec import init_basis

        init_basis(data, self.basis_index(index))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                self._lib.hs_program_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass

    def info(self, i: int) -> dict:
        inf = _native.HsPartInfo()
        _native.check(self._lib.hs_program_part_info(self._h, i, ctypes.byref(inf)))
        return {
            "tile_bits": inf.tile_bits,
            "tile_pos": list(inf.tile_pos[: inf.tile_bits]),
            "reg_bits": inf.reg_bits,
            "phases": inf.phases,
            "instructions": inf.instructions,
            "dense_gates": inf.dense_gates,
            "perm_gates": inf.perm_gates,
            "diag_gates": inf.diag_gates,
            "swaps_relabelled": inf.swaps_relabelled,
            "tiles": inf.tiles,
            "fp_ops_per_amp": inf.fp_ops_per_amp,
            "input_gates": inf.input_gates,
            "restore": bool(inf.restore),
            "compiled": bool(inf.compiled),
            "fp64_instr_per_amp": float(inf.fp64_instr_per_amp),
            "user_part": int(inf.user_part),
        }

    def dump(self, i: int) -> bytes:
        """Raw PartLaunch header + instructions of part i (tests)."""
        count = ctypes.c_int()
        isz = ctypes.c_size_t()
        _native.check(self._lib.hs_program_dump(self._h, i, None, 0, ctypes.byref(count), ctypes.byref(isz)))
        size = 64 + count.value * isz.value + 4096
        buf = ctypes.create_string_buffer(size)
        _native.check(self._lib.hs_program_dump(self._h, i, buf, size, ctypes.byref(count), ctypes.byref(isz)))
        return buf.raw

    def _check(self, data):
        if data.device != self.device or data.dtype != self.dtype:
            raise ValueError(f"state must be {self.dtype} on {self.device}, got {data.dtype} on {data.device}")
        if not data.is_contiguous():
            raise ValueError("state must be C-contiguous")
        rows = data.numel() >> self.n_local
        if rows < 1 or rows << self.n_local != data.numel():
            raise ValueError(f"state of {data.numel()} amplitudes is not rows x 2^{self.n_local}")
        return rows

    def run(self, data, first: int = 0, count: int | None = None, stream=None) -> None:
        """Launch launches [first, first+count) on ``data`` (stream-ordered;
        default: all of them, i.e. every part plus any layout restore)."""
        import torch

        rows = self._check(data)
        count = self.num_launches - first if count is None else count
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._bind_scratch(data)
        _native.check(self._lib.hs_program_run(self._h, data.data_ptr(), rows, first, count, s))

    @property
    def needs_scratch(self) -> bool:
        return bool(self.options & _native.HS_PLAN_PINGPONG)

    def share_scratch(self, scratch) -> None:
        """Use ``scratch`` (a device tensor at least the state's size) as the
        ping-pong partner, e.g. one buffer for several programs."""
        self._scratch = scratch

    def _bind_scratch(self, data) -> None:
        """HS_PLAN_PINGPONG: a device buffer like ``data`` the parts alternate
        with (allocated once per shape, kept by the program)."""
        if not self.options & _native.HS_PLAN_PINGPONG:
            return
        sc = self._scratch
        if sc is None or sc.numel() < data.numel() or sc.dtype != data.dtype or sc.device != data.device:
            import torch

            self._scratch = sc = torch.empty(data.numel(), dtype=data.dtype, device=data.device)
        _native.check(self._lib.hs_program_bind_scratch(self._h, sc.data_ptr(), sc.numel() * sc.element_size()))

    def run_graph(self, data, stream=None) -> None:
        """All parts as one CUDA graph launch (captured on first use)."""
        import torch

        rows = self._check(data)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._bind_scratch(data)
        _native.check(self._lib.hs_program_run_graph(self._h, data.data_ptr(), rows, s))


def _as_device(data):
    """(tensor, writeback) for a numpy or torch buffer."""
    if isinstance(data, np.ndarray):
        if not data.flags.c_contiguous:
            raise ValueError("arr must be C-contiguous")
        import torch

        t = torch.from_numpy(data).to(default_device())

        def back():
            data[...] = t.cpu().numpy()

        return t, back
    return data, None


def run_part(data, exe: ExecutablePart) -> None:
    """One part pass in place on the last axis of ``data`` (hier.py:220-244).

    ``data`` is a contiguous CUDA tensor (complex128/complex64) whose last
    axis has 2^m entries, leading axes batch; every staged position must be
    below m. A numpy array is accepted too (copied to the device and back).
    """
    t, back = _as_device(data)
    last = int(t.shape[-1]) if t.dim() else 1
    m = last.bit_length() - 1
    if last != 1 << m:
        raise ValueError(f"last axis {last} is not a power of two")
    qubits = exe.slot_map.qubits
    if qubits and qubits[-1] >= m:
        raise ValueError(f"position {qubits[-1]} outside 0..{m - 1}")
    if not t.is_contiguous():
        raise ValueError("arr must be C-contiguous")
    if exe.ops:
        _run_part_program(m, exe, t.dtype, t.device).run(t)
    if back is not None:
        back()


#: planned one-part programs of recent ``run_part`` / ``apply_op`` calls: a
#: gate-by-gate caller (apply_gate in a loop, statevec.py:241-266) plans and
#: uploads each distinct (state size, part) once instead of per call
_RUN_PART_CACHE: "dict[tuple, PartProgram]" = {}
RUN_PART_CACHE_SIZE = 256


def _run_part_program(m: int, exe: ExecutablePart, dtype, device) -> "PartProgram":
    key = (m, str(dtype), str(device), exe.slot_map.qubits, exe.ops, exe.op_slots, _native.default_options())
    prog = _RUN_PART_CACHE.pop(key, None)
    if prog is None:
        prog = PartProgram(m, [exe], dtype=dtype, device=device)
        while len(_RUN_PART_CACHE) >= RUN_PART_CACHE_SIZE:
            _RUN_PART_CACHE.pop(next(iter(_RUN_PART_CACHE)))
    _RUN_PART_CACHE[key] = prog  # most recently used last
    return prog


# --- traces ---------------------------------------------------------------------

@dataclass(frozen=True)
class PartTrace:
    """Staging cost of one part (hier.py:249-270); ``time_s``/``hbm_bytes``
    are filled by timed runs (per-part CUDA events), else None."""

    part_id: int
    level: int
    parent_id: int | None
    num_qubits: int
    num_gates: int
    gather_calls: int
    scatter_calls: int
    inner_bytes: int
    time_s: float | None = None
    hbm_bytes: int | None = None


@dataclass
class ExecutionTrace:
    num_qubits: int
    parts: list[PartTrace] = field(default_factory=list)

    @property
    def total_gather_calls(self) -> int:
        return sum(p.gather_calls for p in self.parts)

    @property
    def total_scatter_calls(self) -> int:
        return sum(p.scatter_calls for p in self.parts)

    def level_parts(self, level: int) -> list[PartTrace]:
        return [p for p in self.parts if p.level == level]

    def part_rows(self) -> list[dict]:
        """The reference's row schema (hier.py:287-303), plus timing fields
        when a timed run filled them."""
        rows = []
        for p in self.parts:
            row = {"part_id": p.part_id, "w": p.num_qubits, "iterations": p.gather_calls,
                   "gates": p.num_gates, "level": p.level, "parent_id": p.parent_id}
            if p.time_s is not None:
                row["time_s"] = p.time_s
                row["hbm_bytes"] = p.hbm_bytes
                row["gbps"] = p.hbm_bytes / p.time_s / 1e9 if p.time_s > 0 else None
            rows.append(row)
        return rows

    def to_json_lines(self) -> str:
        return "\n".join(json.dumps(r) for r in self.part_rows())

    def to_json(self) -> dict:
        return {"num_qubits": self.num_qubits, "total_gather_calls": self.total_gather_calls,
                "total_scatter_calls": self.total_scatter_calls, "parts": self.part_rows()}


def _trace_row(n: int, part_id: int, level: int, parent_id, w: int, gates: int) -> PartTrace:
    calls = 1 << (n - w)
    return PartTrace(part_id, level, parent_id, w, gates, calls, calls, 1 << (w + 4))


def hierarchical_trace(circuit: Circuit, partition: PartitionResult) -> ExecutionTrace:
    """Trace rows of ``execute_hierarchical`` (hier.py:363-365)."""
    n = circuit.num_qubits
    tr = ExecutionTrace(n)
    for p in partition.parts:
        tr.parts.append(_trace_row(n, p.id, 1, None, p.working_set, len(p.gate_indices)))
    return tr


def multilevel_trace(circuit: Circuit, partition: MultiLevelPartition) -> ExecutionTrace:
    """Trace rows of ``execute_multilevel`` (hier.py:389-415): a level-1 row
    per parent, then a level-2 row per sub-part unless the sublevel is lone;
    level-2 iterations = 2^(n-w1) blocks x 2^(w1-w2) stagings = 2^(n-w2)."""
    n = circuit.num_qubits
    tr = ExecutionTrace(n)
    for i, parent in enumerate(partition.level1.parts):
        sub = partition.sublevels[i]
        padded = partition.padded_qubits[i]
        tr.parts.append(_trace_row(n, parent.id, 1, None, parent.working_set, len(parent.gate_indices)))
        if len(sub.parts) == 1 and padded[0] == parent.qubits:
            continue
        for j, sp in enumerate(sub.parts):
            tr.parts.append(_trace_row(n, sp.id, 2, parent.id, len(padded[j]), len(sp.gate_indices)))
    return tr


def timed_launches(program: "PartProgram", data, stream=None) -> list[float]:
    """Run every launch of ``program`` on ``data`` one at a time with CUDA
    events between launches on the launch stream; returns the seconds of
    each launch (synchronizes)."""
    import torch

    s = stream or torch.cuda.current_stream(program.device)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(program.num_launches + 1)]
    ev[0].record(s)
    for i in range(program.num_launches):
        program.run(data, i, 1, stream=s)
        ev[i + 1].record(s)
    ev[-1].synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(program.num_launches)]


def launch_times_by_part(program: "PartProgram", launch_s: Sequence[float]) -> dict[int, tuple[float, int]]:
    """{program part index: (seconds, launches)}. A launch carries the gates
    of the part it reports (``user_part``; regrouped tile passes report the
    part that contributes most of their gates); a gate-free layout launch
    (user_part -1) is charged to the part before it (part 0 if first), so
    the parts' times add up to the program's."""
    out: dict[int, list] = {}
    prev = 0
    for i, t in enumerate(launch_s):
        u = program.info(i)["user_part"]
        u = prev if u < 0 else u
        prev = u
        acc = out.setdefault(u, [0.0, 0])
        acc[0] += t
        acc[1] += 1
    return {k: (v[0], v[1]) for k, v in out.items()}


def _timed_trace(trace: "ExecutionTrace", rows: Sequence[int], program: "PartProgram", launch_s) -> "ExecutionTrace":
    """Fill ``time_s`` / ``hbm_bytes`` of trace row ``rows[j]`` from the
    launches of the program's part j (rows without launches: 0 s, 0 B)."""
    from dataclasses import replace

    amp = 16 if str(program.dtype).endswith("complex128") else 8
    per_pass = 2 * (1 << program.n_local) * amp
    got = launch_times_by_part(program, launch_s)
    parts = list(trace.parts)
    for j, r in enumerate(rows):
        t, k = got.get(j, (0.0, 0))
        parts[r] = replace(parts[r], time_s=t, hbm_bytes=k * per_pass)
    trace.parts = parts
    return trace


# --- drivers ----------------------------------------------------------------------

def start_state(circuit: Circuit, initial, max_qubits, dtype="complex128", device=None) -> StateVector:
    """Fresh device state: |0..0> or a copy of ``initial`` (never aliased)."""
    if initial is None:
        return zero_state(circuit.num_qubits, max_qubits, dtype=dtype, device=device)
    if initial.num_qubits != circuit.num_qubits:
        raise ValueError(
            f"initial state has {initial.num_qubits} qubits, circuit has {circuit.num_qubits}"
        )
    if isinstance(initial.data, np.ndarray):
        return from_numpy(initial.data, dtype, device)
    import torch

    dt = torch.complex64 if str(dtype) in ("complex64", "c64", "torch.complex64") else torch.complex128
    return StateVector(initial.num_qubits, initial.data.to(device or default_device(), dt, copy=True).contiguous())


def _check_covers(circuit: Circuit, parts: Sequence[Part]) -> None:
    seen = [g for p in parts for g in p.gate_indices]
    if len(seen) != circuit.num_ops or set(seen) != set(range(circuit.num_ops)):
        raise ValueError("partition does not cover the circuit exactly once")


class HierarchicalRun:
    """Plan once, run many times: the device program of a partitioned
    circuit (the reusable core of ``execute_hierarchical``)."""

    def __init__(self, circuit: Circuit, partition: PartitionResult, dtype="complex128", device=None,
                 options: int | None = None, basis_start: bool = False):
        """``basis_start``: runs start from basis states prepared with
        ``program.init_basis`` (lets the planner choose the initial layout)."""
        _check_covers(circuit, partition.parts)
        self.circuit = circuit
        self.partition = partition
        self.exes = [remap_part(circuit, p) for p in partition.parts]
        self.program = PartProgram(circuit.num_qubits, self.exes, dtype=dtype, device=device, options=options,
                                   basis_start=basis_start)

    def run_stream(self, inputs, outputs, buffers=None, stream=None, copy_streams: int = 1,
                   copy_chunks: int = 4) -> None:
        """Simulate the circuit on a sequence of host states: ``inputs[i]``
        (pinned host tensors, natural order, e.g. many initial states) ->
        ``outputs[i]``. Uploads, passes and downloads run on their own
        streams over three device buffers (by default), so step i + 1's
        upload, step i's passes and step i - 1's download all overlap (with
        two buffers an upload waits for the download before it). Each copy is
        split into ``copy_chunks`` pieces over ``copy_streams`` streams per
        direction (measured on c3, ms per step: 1 stream x 1 piece 440, 1 x 4
        419, 2 x 2 481, 2 x 4 446, 4 x 4 494; the pipeline is PCIe / host
        memory bound at ~41 GB/s each way). Returns when the last download is queued
        (synchronize to read outputs). The program must accept natural-order
        input (``basis_start=False``)."""
        import torch

        if self.program.initial_layout != tuple(range(self.program.n_local)):
            raise ValueError("run_stream needs a program without its own initial layout (basis_start=False)")
        if len(inputs) != len(outputs):
            raise ValueError("inputs and outputs differ in length")
        dev = self.program.device
        compute = stream or torch.cuda.current_stream(dev)
        if buffers is None:
            like = inputs[0]
            buffers = [torch.empty(like.shape, dtype=self.program.dtype, device=dev) for _ in range(3)]
        ups = [torch.cuda.Stream(dev) for _ in range(copy_streams)]
        downs = [torch.cuda.Stream(dev) for _ in range(copy_streams)]
        free = [None for _ in buffers]  # per buffer: events of its last download

        def pieces(t):
            flat = t.reshape(-1)
            step = -(-flat.numel() // copy_chunks)
            return [flat[i:i + step] for i in range(0, flat.numel(), step)]

        for i, (src, dst) in enumerate(zip(inputs, outputs)):
            b = i % len(buffers)
            buf = buffers[b]
            loaded = []
            for j, (d, h) in enumerate(zip(pieces(buf), pieces(src))):
                up = ups[j % copy_streams]
                with torch.cuda.stream(up):
                    for ev in free[b] or ():
                        up.wait_event(ev)  # the buffer's previous result is downloaded
                    d.copy_(h, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(up)
                    loaded.append(ev)
            for ev in loaded:
                compute.wait_event(ev)
            self.program.run(buf, stream=compute)
            done = torch.cuda.Event()
            done.record(compute)
            evs = []
            for j, (h, d) in enumerate(zip(pieces(dst), pieces(buf))):
                down = downs[j % copy_streams]
                with torch.cuda.stream(down):
                    down.wait_event(done)
                    h.copy_(d, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(down)
                    evs.append(ev)
            free[b] = evs
        for evs in free:
            for ev in evs or ():
                compute.wait_event(ev)

    def trace(self) -> ExecutionTrace:
        return hierarchical_trace(self.circuit, self.partition)


def execute_hierarchical(
    circuit: Circuit,
    partition: PartitionResult,
    *,
    initial: StateVector | None = None,
    max_qubits: int | None = None,
    with_trace: bool = False,
    with_timing: bool = False,
    dtype="complex128",
    device=None,
):
    """Run a partitioned circuit part by part on one device state
    (hier.py:342-368): parts in the given order, as planned tile passes.
    Returns a device ``StateVector`` (and the ``ExecutionTrace``).
    ``with_timing`` (with ``with_trace``): launches run one by one between
    CUDA events and each trace row gets ``time_s``, ``hbm_bytes`` (2 x 2^n x
    amplitude size per launch) and ``gbps``."""
    state = start_state(circuit, initial, max_qubits, dtype, device)
    # from |0..0> (one amplitude, the same in every layout) the planner may
    # choose the initial layout; a caller's state arrives in natural order
    run = HierarchicalRun(circuit, partition, dtype=dtype, device=device, basis_start=initial is None)
    if with_trace and with_timing:
        launch_s = timed_launches(run.program, state.data)
        return state, _timed_trace(run.trace(), range(len(run.exes)), run.program, launch_s)
    run.program.run(state.data)
    if with_trace:
        return state, run.trace()
    return state


def execute_multilevel(
    circuit: Circuit,
    partition: MultiLevelPartition,
    *,
    initial: StateVector | None = None,
    max_qubits: int | None = None,
    with_trace: bool = False,
    with_timing: bool = False,
    dtype="complex128",
    device=None,
):
    """Two-level execution (hier.py:371-419). Staging a level-2 part's
    padded set inside the gathered level-1 block touches the same amplitude
    groups as staging that padded set directly in the state, so each
    level-2 part is one pass with its padded qubits staged; a lone sublevel
    runs as its parent. Trace rows follow the reference exactly."""
    _check_covers(circuit, [p for sub in partition.sublevels for p in sub.parts])
    n = circuit.num_qubits
    exes: list[ExecutablePart] = []
    rows: list[int] = []  # trace row of each executed part
    row = 0
    for i, parent in enumerate(partition.level1.parts):
        sub = partition.sublevels[i]
        padded = partition.padded_qubits[i]
        if len(sub.parts) == 1 and padded[0] == parent.qubits:
            exes.append(remap_part(circuit, sub.parts[0]))
            rows.append(row)
            row += 1
            continue
        exes += [remap_part(circuit, sp, stage_qubits=padded[j]) for j, sp in enumerate(sub.parts)]
        rows += [row + 1 + j for j in range(len(sub.parts))]
        row += 1 + len(sub.parts)
    trace = multilevel_trace(circuit, partition)
    state = start_state(circuit, initial, max_qubits, dtype, device)
    if exes:
        prog = PartProgram(n, exes, dtype=dtype, device=device)
        if with_trace and with_timing:
            trace = _timed_trace(trace, rows, prog, timed_launches(prog, state.data))
        else:
            prog.run(state.data)
    if with_trace:
        return state, trace
    return state


#: planner options of the independent gate-by-gate run behind
#: ``simulate_flat`` / ``verify_against_flat``: no single-qubit fusion, no
#: parity diagonals, no pass merging, no compiled kernels, no layouts - the
#: interpreter kernel runs each gate as its own pass in natural order, so a
#: planner or code-generator bug in the hierarchical run cannot verify itself
FLAT_OPTIONS = 0


def flat_program(circuit: Circuit, dtype="complex128", device=None) -> PartProgram:
    """The gate-by-gate device program: one part, and one launch, per gate."""
    exes = []
    for i, op in enumerate(circuit.ops):
        staged = tuple(sorted(op.qubits))
        exes.append(ExecutablePart(i, (i,), QubitSlotMap(staged), (op,),
                                   (tuple(staged.index(q) for q in op.qubits),)))
    return PartProgram(circuit.num_qubits, exes, dtype=dtype, device=device, options=FLAT_OPTIONS)


def execute_parts_as_gates(circuit: Circuit, max_qubits=None, dtype="complex128", device=None) -> StateVector:
    """Every gate as its own pass (``simulate_flat`` on the device,
    statevec.py:269-277): ``FLAT_OPTIONS``, one interpreter launch per gate."""
    state = zero_state(circuit.num_qubits, max_qubits, dtype=dtype, device=device)
    if circuit.ops:
        prog = flat_program(circuit, dtype=dtype, device=device)
        assert prog.num_launches == circuit.num_ops
        prog.run(state.data)
    return state


def max_abs_diff(state: StateVector, expect) -> float:
    """max |state - expect| on the device (hs_max_abs_diff); ``expect`` is a
    complex128 array/tensor in natural order."""
    import torch

    lib = _native.load()
    if isinstance(expect, StateVector):
        expect = expect.data
    if isinstance(expect, np.ndarray):
        expect = torch.from_numpy(np.ascontiguousarray(expect, dtype=np.complex128)).to(state.data.device)
    expect = expect.to(state.data.device, torch.complex128).contiguous()
    if expect.numel() != state.data.numel():
        raise ValueError("states differ in size")
    out = ctypes.c_double()
    s = torch.cuda.current_stream(state.data.device).cuda_stream
    _native.check(lib.hs_max_abs_diff(state.data.data_ptr(), native_dtype(state.data), expect.data_ptr(),
                                      state.data.numel(), ctypes.byref(out), s))
    return out.value


def verify_against_flat(circuit: Circuit, state: StateVector, atol: float = 1e-10) -> float:
    """Compare with the independent gate-by-gate device run (hier.py:422-436;
    ``FLAT_OPTIONS``: one interpreter pass per gate, none of the planner's
    merging, fusion, layouts or compiled kernels); raises
    ``VerificationError`` above ``atol``."""
    ref = execute_parts_as_gates(circuit, max_qubits=state.num_qubits, dtype=state.data.dtype,
                                 device=state.data.device)
    err = max_abs_diff(state, ref.data.to(dtype=__import__("torch").complex128))
    if not err <= atol:
        raise VerificationError(f"max amplitude deviation {err:.3e} exceeds {atol:.1e}")
    return err
