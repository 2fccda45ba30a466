"""Device state vectors and single-gate application.

API mirror of ``hisim.statevec`` (/root/reference/pkg/src/hisim/statevec.py):
``StateVector``, ``state_bytes``, ``max_qubits_cap``, ``zero_state``,
``gate_matrix``, ``apply_op``, ``apply_gate``, ``simulate_flat``,
``save_state``/``load_state``. The amplitudes live in HBM as a torch CUDA
tensor (complex128 by default, complex64 optional); every arithmetic step
runs in libhisvsim.so (include/hisvsim.h). Little-endian indexing as in the
reference: bit i of a basis index is qubit i.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import DeviceError, QubitCountOutOfRangeError
from .qasm import Circuit, GateKind, GateOp

#: The reference caps host materialization at 24 qubits unless
#: HISIM_MAX_QUBITS raises it (statevec.py:26-29) to stop accidental 16 GiB
#: numpy allocations. On the device the binding limit is free HBM, checked
#: in ``allocate``; the default cap is therefore the hard ceiling, and the
#: env var / ``max_qubits`` argument still lower it like in the reference.
HARD_MAX_QUBITS = 36
DEFAULT_MAX_QUBITS = HARD_MAX_QUBITS

_R2 = 1.0 / math.sqrt(2.0)


def _rx(t):
    c, s = math.cos(t / 2), math.sin(t / 2)
    return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)


def _ry(t):
    c, s = math.cos(t / 2), math.sin(t / 2)
    return np.array([[c, -s], [s, c]], dtype=np.complex128)


def _rz(t):
    return np.array([[np.exp(-0.5j * t), 0], [0, np.exp(0.5j * t)]], dtype=np.complex128)


def _u1(lam):
    return np.array([[1, 0], [0, np.exp(1j * lam)]], dtype=np.complex128)


def _u3(t, phi, lam):
    c, s = math.cos(t / 2), math.sin(t / 2)
    return np.array(
        [[c, -np.exp(1j * lam) * s], [np.exp(1j * phi) * s, np.exp(1j * (phi + lam)) * c]],
        dtype=np.complex128,
    )


_FIXED = {
    GateKind.H: np.array([[_R2, _R2], [_R2, -_R2]], dtype=np.complex128),
    GateKind.X: np.array([[0, 1], [1, 0]], dtype=np.complex128),
    GateKind.Y: np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    GateKind.Z: np.array([[1, 0], [0, -1]], dtype=np.complex128),
    GateKind.S: np.array([[1, 0], [0, 1j]], dtype=np.complex128),
    GateKind.SDG: np.array([[1, 0], [0, -1j]], dtype=np.complex128),
    GateKind.T: np.array([[1, 0], [0, np.exp(0.25j * np.pi)]], dtype=np.complex128),
    GateKind.TDG: np.array([[1, 0], [0, np.exp(-0.25j * np.pi)]], dtype=np.complex128),
}
_PARAMETRIC = {GateKind.RX: _rx, GateKind.RY: _ry, GateKind.RZ: _rz, GateKind.U1: _u1, GateKind.U3: _u3}
#: controlled kind -> (kind of the 2x2 on the target, number of controls)
CONTROLLED = {
    GateKind.CX: (GateKind.X, 1),
    GateKind.CZ: (GateKind.Z, 1),
    GateKind.CRZ: (GateKind.RZ, 1),
    GateKind.CRY: (GateKind.RY, 1),
    GateKind.CCX: (GateKind.X, 2),
}


def base_matrix(kind: GateKind, params: tuple[float, ...] = ()) -> np.ndarray:
    """The 2x2 on the target (controls act by masking); statevec.py:92-98."""
    kind = CONTROLLED.get(kind, (kind, 0))[0]
    if kind in _FIXED:
        return _FIXED[kind]
    return _PARAMETRIC[kind](*params)


def gate_matrix(kind: GateKind, params: tuple[float, ...] = ()) -> np.ndarray:
    """Full 2^arity unitary, first operand = most significant matrix bit
    (statevec.py:101-119). Host-side helper for tests and tooling."""
    if kind is GateKind.SWAP:
        return np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]
    if kind in CONTROLLED:
        _, nc = CONTROLLED[kind]
        dim = 1 << (nc + 1)
        m = np.eye(dim, dtype=np.complex128)
        m[dim - 2:, dim - 2:] = base_matrix(kind, params)
        return m
    return base_matrix(kind, params).copy()


# --- device state -----------------------------------------------------------

def _torch():
    import torch

    return torch


def _dtype_of(name):
    torch = _torch()
    if name in (None, "complex128", "c128", torch.complex128):
        return torch.complex128
    if name in ("complex64", "c64", torch.complex64):
        return torch.complex64
    raise ValueError(f"unsupported dtype {name!r} (complex128 or complex64)")


def native_dtype(t) -> int:
    """C-ABI dtype code of a torch tensor."""
    torch = _torch()
    if t.dtype == torch.complex128:
        return 0
    if t.dtype == torch.complex64:
        return 1
    raise ValueError(f"state tensor must be complex128 or complex64, got {t.dtype}")


def default_device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the engine runs on B200 only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class StateVector:
    """2^n amplitudes in HBM (``data`` is a CUDA tensor, natural order)."""

    num_qubits: int
    data: "object"

    def norm(self) -> float:
        return float(_torch().linalg.vector_norm(self.data).item())

    def copy(self) -> "StateVector":
        return StateVector(self.num_qubits, self.data.clone())

    def to_numpy(self) -> np.ndarray:
        """Host copy as complex128 (the reference's representation)."""
        return self.data.detach().cpu().numpy().astype(np.complex128, copy=False)

    @property
    def dtype(self):
        return self.data.dtype


def state_bytes(n: int, dtype="complex128") -> int:
    """Footprint of an n-qubit vector: 2^(n+4) bytes for complex128,
    2^(n+3) for complex64 (statevec.py:138-140)."""
    return 1 << (n + (3 if str(dtype) in ("complex64", "c64", "torch.complex64") else 4))


def max_qubits_cap(max_qubits: int | None = None) -> int:
    """Argument, else ``HISIM_MAX_QUBITS``, else the default, capped at
    ``HARD_MAX_QUBITS`` (statevec.py:143-148)."""
    if max_qubits is None:
        env = os.environ.get("HISIM_MAX_QUBITS")
        max_qubits = int(env) if env else DEFAULT_MAX_QUBITS
    return min(max_qubits, HARD_MAX_QUBITS)


def free_bytes(device) -> int:
    """Free HBM on ``device`` as allocations see it: the driver's free memory
    plus what torch's caching allocator holds reserved but unused."""
    torch = _torch()
    free, _ = torch.cuda.mem_get_info(device)
    return free + torch.cuda.memory_reserved(device) - torch.cuda.memory_allocated(device)


def allocate(n: int, dtype="complex128", device=None, rows: int = 1):
    """Uninitialized device buffer of rows x 2^n amplitudes; raises
    ``QubitCountOutOfRangeError`` if it does not fit in free HBM."""
    torch = _torch()
    dt = _dtype_of(dtype)
    device = device or default_device()
    need = rows * (1 << n) * (16 if dt == torch.complex128 else 8)
    free = free_bytes(device)
    if need > free:
        raise QubitCountOutOfRangeError(
            f"{need} bytes for {rows} x 2^{n} amplitudes exceed {free} free bytes on {device}"
        )
    return torch.empty((rows, 1 << n) if rows > 1 else (1 << n,), dtype=dt, device=device)


def init_basis(data, index: int = 0) -> None:
    """Set a device buffer to the basis state |index> (hs_state_init_basis)."""
    from . import _native

    lib = _native.load()
    stream = _torch().cuda.current_stream(data.device).cuda_stream
    _native.check(lib.hs_state_init_basis(data.data_ptr(), data.numel(), native_dtype(data), index, stream))


def zero_state(n: int, max_qubits: int | None = None, dtype="complex128", device=None) -> StateVector:
    """|0...0> on the device. Refuses n outside [1, cap] like the reference
    (statevec.py:151-167); the cap is ``max_qubits_cap``."""
    cap = max_qubits_cap(max_qubits)
    if not 1 <= n <= cap:
        detail = f", {state_bytes(n)} bytes" if n >= 1 else ""
        raise QubitCountOutOfRangeError(
            f"n={n} outside [1, {cap}] (cap from HISIM_MAX_QUBITS or max_qubits, "
            f"ceiling {HARD_MAX_QUBITS}{detail})"
        )
    data = allocate(n, dtype, device)
    init_basis(data, 0)
    return StateVector(n, data)


def from_numpy(arr: np.ndarray, dtype="complex128", device=None) -> StateVector:
    """Upload a host amplitude array (natural order)."""
    torch = _torch()
    n = int(arr.size).bit_length() - 1
    if arr.size != 1 << n:
        raise ValueError(f"{arr.size} amplitudes is not a power of two")
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.complex128))
    return StateVector(n, t.to(device or default_device()).to(_dtype_of(dtype)))


# --- gates ------------------------------------------------------------------

def apply_op(arr, w: int, op: GateOp, slots: tuple[int, ...] | None = None) -> None:
    """Apply one gate in place to every w-qubit block of ``arr`` (last axis
    2^w, leading axes batch); statevec.py:241-261. ``arr`` is a contiguous
    CUDA tensor. Runs as a one-gate part through hs_part_apply."""
    from .hier import ExecutablePart, QubitSlotMap, run_part

    if not arr.is_contiguous():
        raise ValueError("arr must be C-contiguous")
    q = tuple(slots) if slots is not None else tuple(op.qubits)
    staged = tuple(sorted(q))
    exe = ExecutablePart(-1, (), QubitSlotMap(staged), (op,), (tuple(staged.index(x) for x in q),))
    run_part(arr, exe)


def apply_gate(state: StateVector, op: GateOp) -> None:
    """Apply one gate to a full device state in place."""
    apply_op(state.data, state.num_qubits, op)


def simulate_flat(circuit: Circuit, max_qubits: int | None = None, dtype="complex128") -> StateVector:
    """Gate-by-gate simulation on the device (statevec.py:269-277): every
    gate is its own interpreter pass with the planner's merging, fusion,
    layouts and code generation off (``hier.FLAT_OPTIONS``), so it is
    independent of the hierarchical path it verifies. The parity oracle of
    the test suite is the CPU restatement under ``oracle/``, not this."""
    from .hier import execute_parts_as_gates

    return execute_parts_as_gates(circuit, max_qubits=max_qubits, dtype=dtype)


# --- dumps --------------------------------------------------------------------

def save_state(state: StateVector, path) -> None:
    """Little-endian complex128 dump plus ``<path>.json`` sidecar
    {num_qubits, norm} (statevec.py:282-288)."""
    path = Path(path)
    host = state.to_numpy()
    host.astype("<c16").tofile(path)
    side = {"num_qubits": state.num_qubits, "norm": float(np.linalg.norm(host))}
    Path(str(path) + ".json").write_text(json.dumps(side, indent=2) + "\n")


def load_state(path, dtype="complex128", device=None) -> StateVector:
    """Read a ``save_state`` dump onto the device, checking its size."""
    path = Path(path)
    meta = json.loads(Path(str(path) + ".json").read_text())
    n = int(meta["num_qubits"])
    data = np.fromfile(path, dtype="<c16")
    if data.size != 1 << n:
        raise ValueError(f"dump holds {data.size} amplitudes, expected {1 << n}")
    return from_numpy(data, dtype, device)
