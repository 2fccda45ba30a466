"""CPU oracle: numpy restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY. Imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs, always as
the checker or the timed CPU baseline, never as part of the product path
(the package ``paper_2205_06973_b200`` never imports it).

Pinned: every function here is checked against golden vectors produced by
the reference package itself (``tests/golden/make_golden.py`` imports
/root/reference/pkg/src/hisim and writes ``tests/golden/*.json|npz``) and
against the reference's own known-answer tests.

Each function restates the reference algorithm it cites; gate circuits use
the package's IR (``GateKind``/``GateOp``/``Circuit``) so the same circuit
objects feed the oracle and the device engine.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2205_06973_b200.qasm import Circuit, GateKind, GateOp

# --- gate matrices, restated from statevec.py:31-98 (independent of the
# package's own tables so a wrong entry there cannot hide) -------------------

_S2 = 1.0 / math.sqrt(2.0)
_FIXED = {
    GateKind.H: [[_S2, _S2], [_S2, -_S2]],
    GateKind.X: [[0, 1], [1, 0]],
    GateKind.Y: [[0, -1j], [1j, 0]],
    GateKind.Z: [[1, 0], [0, -1]],
    GateKind.S: [[1, 0], [0, 1j]],
    GateKind.SDG: [[1, 0], [0, -1j]],
    GateKind.T: [[1, 0], [0, np.exp(0.25j * np.pi)]],
    GateKind.TDG: [[1, 0], [0, np.exp(-0.25j * np.pi)]],
}
#: controlled kind -> (2x2 kind on the target, number of controls)
CONTROLLED = {
    GateKind.CX: (GateKind.X, 1),
    GateKind.CZ: (GateKind.Z, 1),
    GateKind.CRZ: (GateKind.RZ, 1),
    GateKind.CRY: (GateKind.RY, 1),
    GateKind.CCX: (GateKind.X, 2),
}


def base_matrix(kind: GateKind, params=()) -> np.ndarray:
    """The 2x2 acting on the target (statevec.py:92-98)."""
    kind = CONTROLLED.get(kind, (kind, 0))[0]
    if kind in _FIXED:
        return np.array(_FIXED[kind], dtype=np.complex128)
    t = params[0]
    c, s = math.cos(t / 2), math.sin(t / 2)
    if kind is GateKind.RX:
        m = [[c, -1j * s], [-1j * s, c]]
    elif kind is GateKind.RY:
        m = [[c, -s], [s, c]]
    elif kind is GateKind.RZ:
        m = [[np.exp(-0.5j * t), 0], [0, np.exp(0.5j * t)]]
    elif kind is GateKind.U1:
        m = [[1, 0], [0, np.exp(1j * t)]]
    else:  # U3(theta, phi, lambda)
        phi, lam = params[1], params[2]
        m = [[c, -np.exp(1j * lam) * s], [np.exp(1j * phi) * s, np.exp(1j * (phi + lam)) * c]]
    return np.array(m, dtype=np.complex128)


# --- statevec.py:172-261 ----------------------------------------------------

def apply_1q(arr: np.ndarray, u: np.ndarray, t: int) -> None:
    """2x2 on slot t of every block (statevec.py:172-185): pairs at stride
    2^t; a diagonal u only scales the non-unit halves."""
    v = arr.reshape(-1, 2, 1 << t)
    lo, hi = v[:, 0, :], v[:, 1, :]
    if u[0, 1] == 0 and u[1, 0] == 0:
        if u[0, 0] != 1.0:
            lo *= u[0, 0]
        if u[1, 1] != 1.0:
            hi *= u[1, 1]
        return
    new_lo = u[0, 0] * lo + u[0, 1] * hi
    v[:, 1, :] = u[1, 0] * lo + u[1, 1] * hi
    v[:, 0, :] = new_lo


def apply_controlled(arr: np.ndarray, w: int, u: np.ndarray, t: int, controls) -> None:
    """2x2 on slot t where every control slot is 1 (statevec.py:188-225)."""
    rows = arr.size >> w
    cube = arr.reshape((rows,) + (2,) * w)  # axis 1 + (w-1-s) is slot s
    sel = [slice(None)] * (w + 1)
    for c in controls:
        sel[w - c] = 1
    view = cube[tuple(sel)]
    axis = w - t - sum(1 for c in controls if c > t)
    m = np.moveaxis(view, axis, 0)
    lo, hi = m[0], m[1]
    if u[0, 1] == 0 and u[1, 0] == 0:
        if u[0, 0] != 1.0:
            lo *= u[0, 0]
        if u[1, 1] != 1.0:
            hi *= u[1, 1]
        return
    new_lo = u[0, 0] * lo + u[0, 1] * hi
    m[1] = u[1, 0] * lo + u[1, 1] * hi
    m[0] = new_lo


def apply_swap(arr: np.ndarray, w: int, a: int, b: int) -> None:
    """Exchange the 01 and 10 sub-blocks of slots (a, b) (statevec.py:228-238)."""
    rows = arr.size >> w
    cube = arr.reshape((rows,) + (2,) * w)
    s01 = [slice(None)] * (w + 1)
    s10 = [slice(None)] * (w + 1)
    s01[w - a], s01[w - b] = 0, 1
    s10[w - a], s10[w - b] = 1, 0
    keep = cube[tuple(s01)].copy()
    cube[tuple(s01)] = cube[tuple(s10)]
    cube[tuple(s10)] = keep


def apply_op(arr: np.ndarray, w: int, op: GateOp, slots=None) -> None:
    """Dispatch one gate onto every w-slot block of ``arr`` in place
    (statevec.py:241-261)."""
    if not arr.flags.c_contiguous:
        raise ValueError("arr must be C-contiguous")
    q = tuple(slots) if slots is not None else op.qubits
    if op.kind is GateKind.SWAP:
        apply_swap(arr, w, q[0], q[1])
        return
    u = base_matrix(op.kind, op.params)
    if op.kind in CONTROLLED:
        nc = CONTROLLED[op.kind][1]
        apply_controlled(arr, w, u, q[nc], q[:nc])
    else:
        apply_1q(arr, u, q[0])


def zero_state(n: int) -> np.ndarray:
    """|0...0> (statevec.py:151-167), no size cap (the oracle is bounded by
    host RAM, callers keep n small)."""
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[0] = 1.0
    return psi


def simulate_flat(circuit: Circuit, initial: np.ndarray | None = None) -> np.ndarray:
    """Every gate in program order on |0..0> (statevec.py:269-277)."""
    psi = zero_state(circuit.num_qubits) if initial is None else np.array(initial, dtype=np.complex128)
    for op in circuit.ops:
        apply_op(psi, circuit.num_qubits, op)
    return psi


# --- hier.py:80-244, 342-419 ---------------------------------------------------

def bit_offsets(bits) -> np.ndarray:
    """hier.py:80-91."""
    k = np.arange(1 << len(bits), dtype=np.int64)
    out = np.zeros_like(k)
    for j, b in enumerate(bits):
        out += ((k >> j) & 1) << b
    return out


def block_indices(m: int, qubits) -> np.ndarray:
    """hier.py:94-109: rows = free fixings, columns = inner index."""
    inside = set(qubits)
    free = [q for q in range(m) if q not in inside]
    return bit_offsets(free)[:, None] + bit_offsets(list(qubits))[None, :]


def run_part(data: np.ndarray, positions, ops, op_slots) -> None:
    """Gather -> gates -> scatter over the last axis (hier.py:220-244)."""
    m = int(data.shape[-1]).bit_length() - 1
    w = len(positions)
    if tuple(positions) == tuple(range(m)):
        for op, sl in zip(ops, op_slots):
            apply_op(data, w, op, sl)
        return
    idx = block_indices(m, positions)
    block = np.ascontiguousarray(data[..., idx])
    for op, sl in zip(ops, op_slots):
        apply_op(block, w, op, sl)
    data[..., idx] = block


def part_slots(circuit: Circuit, gate_indices, staged, position_of=None):
    """(positions, ops, op_slots) like remap_part (hier.py:181-217)."""
    pos_of = (lambda q: q) if position_of is None else (lambda q: position_of[q])
    positions = tuple(sorted(pos_of(q) for q in staged))
    ops = tuple(circuit.ops[g] for g in gate_indices)
    slots = tuple(tuple(positions.index(pos_of(q)) for q in op.qubits) for op in ops)
    return positions, ops, slots


def execute_hierarchical(circuit: Circuit, parts, initial=None) -> np.ndarray:
    """Parts in order, one batched pass each (hier.py:342-368). ``parts`` is a
    sequence of (gate_indices, qubits)."""
    psi = zero_state(circuit.num_qubits) if initial is None else np.array(initial, dtype=np.complex128)
    for gates, qubits in parts:
        run_part(psi, *part_slots(circuit, gates, qubits))
    return psi


def execute_multilevel(circuit: Circuit, level1, sublevels, padded, initial=None) -> np.ndarray:
    """hier.py:371-419: gather each level-1 block once, run its level-2
    parts on padded sets inside it, scatter back."""
    n = circuit.num_qubits
    psi = zero_state(n) if initial is None else np.array(initial, dtype=np.complex128)
    for (pg, pq), subs, pads in zip(level1, sublevels, padded):
        if len(subs) == 1 and tuple(pads[0]) == tuple(pq):
            run_part(psi, *part_slots(circuit, subs[0][0], subs[0][1]))
            continue
        inner = {q: s for s, q in enumerate(sorted(pq))}
        idx = block_indices(n, sorted(pq))
        block = psi[idx]
        for (sg, _sq), pad in zip(subs, pads):
            run_part(block, *part_slots(circuit, sg, pad, position_of=inner))
        psi[idx] = block
    return psi


# --- dist.py:53-166, 271-313, 485-529 ------------------------------------------------

def address_of(local, process, g: int):
    """(rank, offset) of global index g (dist.py:103-111)."""
    off = sum(((g >> q) & 1) << j for j, q in enumerate(local))
    rank = sum(((g >> q) & 1) << k for k, q in enumerate(process))
    return rank, off


def choose_layout(n: int, p: int, part_qubits):
    """Part qubits plus the lowest others as locals (dist.py:126-148)."""
    l = n - p
    local = set(part_qubits)
    for q in range(n):
        if len(local) == l:
            break
        local.add(q)
    return tuple(sorted(local)), tuple(q for q in range(n) if q not in local)


def layout_positions(n: int, local, process) -> np.ndarray:
    """Storage position of every global index (dist.py:151-166)."""
    g = np.arange(1 << n, dtype=np.int64)
    off = np.zeros_like(g)
    for j, q in enumerate(local):
        off |= ((g >> q) & 1) << j
    rank = np.zeros_like(g)
    for k, q in enumerate(process):
        rank |= ((g >> q) & 1) << k
    return (rank << len(local)) | off


def plan_stats(n: int, old, new, bytes_per_amp: int = 16) -> dict:
    """Runs / messages / bytes of a layout switch, by enumerating every
    amplitude's (src rank, src offset) -> (dst rank, dst offset) in source
    order like plan_redistribution (dist.py:271-313)."""
    (ol, op), (nl, nproc) = old, new
    l = len(ol)
    src = layout_positions(n, ol, op)
    dst = layout_positions(n, nl, nproc)
    inv = np.empty_like(src)
    inv[src] = np.arange(1 << n, dtype=np.int64)
    dpos = dst[inv]
    s = np.arange(1 << n, dtype=np.int64)
    srank, drank = s >> l, dpos >> l
    if len(s) > 1:
        brk = (np.diff(srank) != 0) | (np.diff(drank) != 0) | (np.diff(dpos) != 1)
        starts = np.concatenate(([0], np.flatnonzero(brk) + 1))
    else:
        starts = np.array([0])
    ends = np.concatenate((starts[1:], [len(s)]))
    length = ends - starts
    rs, rd = srank[starts], drank[starts]
    remote = rs != rd
    R = 1 << len(op)
    sent = np.bincount(rs[remote], weights=length[remote], minlength=R)
    recv = np.bincount(rd[remote], weights=length[remote], minlength=R)
    return {
        "runs": int(len(starts)),
        "messages": int(len(np.unique(rs[remote] * R + rd[remote]))),
        "bytes_remote": int(bytes_per_amp * length[remote].sum()),
        "bytes_resident": int(bytes_per_amp * length[~remote].sum()),
        "sent_bytes": {r: int(bytes_per_amp * c) for r, c in enumerate(sent) if c},
        "received_bytes": {r: int(bytes_per_amp * c) for r, c in enumerate(recv) if c},
    }


def simulate_distributed(circuit: Circuit, parts, p: int, initial=None):
    """Emulated ranks (dist.py:485-529): returns (state in natural order,
    list of per-switch stats dicts with from/to, list of layouts)."""
    n = circuit.num_qubits
    full = zero_state(n) if initial is None else np.array(initial, dtype=np.complex128)
    layout = choose_layout(n, p, parts[0][1])
    flat = np.empty_like(full)
    flat[layout_positions(n, *layout)] = full
    bufs = flat.reshape(1 << p, -1)
    switches, layouts = [], []
    for i, (gates, qubits) in enumerate(parts):
        if not set(qubits) <= set(layout[0]):
            new = choose_layout(n, p, qubits)
            st = plan_stats(n, layout, new)
            st.update({"from": i - 1, "to": i})
            switches.append(st)
            moved = np.empty_like(flat)
            moved[layout_positions(n, *new)] = bufs.reshape(-1)[layout_positions(n, *layout)]
            flat = moved
            bufs = flat.reshape(1 << p, -1)
            layout = new
        layouts.append(layout)
        pos = {q: j for j, q in enumerate(layout[0])}
        run_part(bufs, *part_slots(circuit, gates, qubits, position_of=pos))
    out = bufs.reshape(-1)[layout_positions(n, *layout)]
    return np.ascontiguousarray(out), switches, layouts


# --- closed forms used at sizes the oracle cannot materialize --------------------------

def qft_basis_amplitudes(n: int, x: int, ks: np.ndarray) -> np.ndarray:
    """Amplitudes a_k of the reference QFT circuit (bench.py:124-135: H +
    crz/u1 controlled phases + final bit-reversal swaps) applied to |x>:
    a_k = 2^(-n/2) exp(2 pi i (rev(x) * rev(k) mod 2^n) / 2^n)
    (SURVEY.md §7.3 hard part 4(b)), in exact integer arithmetic."""
    N = 1 << n

    def rev(v):
        out = 0
        for b in range(n):
            out |= ((v >> b) & 1) << (n - 1 - b)
        return out

    rx = rev(int(x))
    ph = np.array([(rx * rev(int(k))) % N for k in ks], dtype=np.float64)
    return np.exp(2j * math.pi * ph / N) / math.sqrt(N)
