"""ctypes front of the C oracle (oracle/sv_oracle.c -> oracle/_build/libsv_oracle.so).

TEST INFRASTRUCTURE ONLY (see sv_oracle.c): the multi-threaded CPU checker
for sizes the numpy restatement is too slow for, and the timed CPU baseline
of bench.py. Built by ``make -C oracle`` (called from __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2205_06973_b200.qasm import Circuit, GateKind

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libsv_oracle.so"
_KIND = {k: i for i, k in enumerate(GateKind)}


class OrGate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("num_slots", ctypes.c_int32), ("slots", ctypes.c_int32 * 3),
                ("reserved", ctypes.c_int32), ("params", ctypes.c_double * 3)]


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", os.fspath(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(os.fspath(LIB))
        L.or_run_part.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int32),
                                  ctypes.c_int, ctypes.POINTER(OrGate), ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
        L.or_run_part.restype = ctypes.c_int
        L.or_simulate_flat.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(OrGate), ctypes.c_int]
        L.or_simulate_flat.restype = ctypes.c_int
        L.or_num_threads.restype = ctypes.c_int
        L.or_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def threads() -> int:
    return lib().or_num_threads()


def set_threads(t: int) -> None:
    lib().or_set_threads(t)


def _gates(ops, slots):
    arr = (OrGate * max(1, len(ops)))()
    for g, (op, sl) in enumerate(zip(ops, slots)):
        arr[g].kind = _KIND[op.kind]
        arr[g].num_slots = len(sl)
        for a, s in enumerate(sl):
            arr[g].slots[a] = s
        for a, v in enumerate(op.params):
            arr[g].params[a] = float(v)
    return arr


def run_part(data: np.ndarray, positions, ops, slots, fix_begin: int = 0, fix_count: int = -1) -> None:
    """In-place part pass on a complex128 array (last axis 2^m, rows = the
    rest); optionally only fixings [fix_begin, fix_begin + fix_count)."""
    if data.dtype != np.complex128 or not data.flags.c_contiguous:
        raise ValueError("complex128 C-contiguous array required")
    m = int(data.shape[-1]).bit_length() - 1
    rows = data.size >> m
    pos = (ctypes.c_int32 * max(1, len(positions)))(*positions)
    rc = lib().or_run_part(data.ctypes.data, m, rows, pos, len(positions), _gates(ops, slots), len(ops),
                           fix_begin, fix_count)
    if rc:
        raise RuntimeError(f"or_run_part failed ({rc})")


def part_slots(circuit: Circuit, gate_indices, staged):
    positions = tuple(sorted(staged))
    ops = tuple(circuit.ops[g] for g in gate_indices)
    slots = tuple(tuple(positions.index(q) for q in op.qubits) for op in ops)
    return positions, ops, slots


def execute_parts(circuit: Circuit, parts, initial: np.ndarray | None = None) -> np.ndarray:
    """execute_hierarchical over (gate_indices, qubits) parts."""
    n = circuit.num_qubits
    if initial is None:
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[0] = 1.0
    else:
        psi = np.array(initial, dtype=np.complex128)
    for gates, qubits in parts:
        run_part(psi, *part_slots(circuit, gates, qubits))
    return psi


def simulate_flat(circuit: Circuit) -> np.ndarray:
    n = circuit.num_qubits
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[0] = 1.0
    slots = tuple(op.qubits for op in circuit.ops)
    rc = lib().or_simulate_flat(psi.ctypes.data, n, _gates(circuit.ops, slots), len(circuit.ops))
    if rc:
        raise RuntimeError(f"or_simulate_flat failed ({rc})")
    return psi
