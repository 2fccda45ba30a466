"""Seeded generators for the BASELINE.json workloads.

All circuits use the reference's 19-kind gate set (qasm.py:26-47) so the
CPU oracle and the reference run the very same op lists:

* sqrt(X) = U3(pi/2, -pi/2, pi/2), sqrt(Y) = U3(pi/2, 0, 0),
  sqrt(W) = U3(pi/2, -pi/4, pi/4) -- each exact up to the global phase
  e^{i pi/4}, identical on both sides;
* RZZ(theta) = CX(a,b) . RZ(b, theta) . CX(a,b);
* controlled phase CP(lambda) = CRZ(lambda) then U1(lambda/2) on the control,
  the reference's own QFT convention (bench.py:124-135).

The configs stand in for the paper's QASMBench circuits, which are not in
this environment; they are synthetic, seeded, and documented in DESIGN.md.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass

from .qasm import Circuit, GateKind, GateOp

_PI = math.pi
SQRT_X = (_PI / 2, -_PI / 2, _PI / 2)
SQRT_Y = (_PI / 2, 0.0, 0.0)
SQRT_W = (_PI / 2, -_PI / 4, _PI / 4)


def _op(kind, *qubits, params=()):
    return GateOp(kind, tuple(qubits), tuple(float(p) for p in params))


def qft_config(n: int = 20, seed: int = 0) -> Circuit:
    """c1: X on a seeded subset (random() < 0.5 per qubit), then the QFT of
    bench.qft: H(i); for j > i: CRZ(j->i, pi/2^(j-i)), U1(j, pi/2^(j-i+1));
    then SWAP(i, n-1-i) for i < n/2."""
    rng = random.Random(seed)
    ops = [_op(GateKind.X, q) for q in range(n) if rng.random() < 0.5]
    for i in range(n):
        ops.append(_op(GateKind.H, i))
        for j in range(i + 1, n):
            theta = _PI / (1 << (j - i))
            ops.append(_op(GateKind.CRZ, j, i, params=(theta,)))
            ops.append(_op(GateKind.U1, j, params=(theta / 2,)))
    ops += [_op(GateKind.SWAP, i, n - 1 - i) for i in range(n // 2)]
    return Circuit(n, tuple(ops))


def qft_prefix_index(n: int = 20, seed: int = 0) -> int:
    """The basis index |x> the c1 X-prefix prepares."""
    rng = random.Random(seed)
    return sum(1 << q for q in range(n) if rng.random() < 0.5)


def grid_patterns(rows: int, cols: int, sites: dict[tuple[int, int], int]):
    """8 cyclic CZ patterns over grid edges: {horizontal, vertical} x
    {edge offset 0,1} x {row/column parity 0,1}; every pattern is a matching."""
    pats = []
    for horizontal in (True, False):
        for off in (0, 1):
            for par in (0, 1):
                edges = []
                for r in range(rows):
                    for c in range(cols):
                        if horizontal:
                            a, b = (r, c), (r, c + 1)
                            ok = c % 2 == off and r % 2 == par
                        else:
                            a, b = (r, c), (r + 1, c)
                            ok = r % 2 == off and c % 2 == par
                        if ok and a in sites and b in sites:
                            edges.append((sites[a], sites[b]))
                pats.append(edges)
    return pats


def random_grid_circuit(rows: int, cols: int, depth: int, seed: int,
                        drop: tuple[tuple[int, int], ...] = (), extra_at: tuple[int, int] | None = None) -> Circuit:
    """Supremacy-style circuit (c2/c5): per layer a seeded sqrt(X)/sqrt(Y)/
    sqrt(W) on every qubit (never the same gate twice in a row on a qubit),
    then CZ on grid pattern ``layer % 8``. ``drop`` removes grid sites;
    ``extra_at`` attaches one more qubit to that site, its CZ joining every
    pattern in which the site is otherwise idle."""
    sites = {}
    for r in range(rows):
        for c in range(cols):
            if (r, c) not in drop:
                sites[(r, c)] = len(sites)
    n = len(sites)
    pats = grid_patterns(rows, cols, sites)
    if extra_at is not None:
        anchor = sites[extra_at]
        for p in pats:
            if all(anchor not in e for e in p):
                p.append((anchor, n))
        n += 1
    rng = random.Random(seed)
    choices = (SQRT_X, SQRT_Y, SQRT_W)
    last = [None] * n
    ops = []
    for layer in range(depth):
        for q in range(n):
            opts = [g for g in range(3) if g != last[q]]
            g = rng.choice(opts)
            last[q] = g
            ops.append(_op(GateKind.U3, q, params=choices[g]))
        for a, b in pats[layer % 8]:
            ops.append(_op(GateKind.CZ, a, b))
    return Circuit(n, tuple(ops))


def random_3_regular(n: int, rng: random.Random) -> list[tuple[int, int]]:
    """Seeded simple 3-regular graph by the configuration model with retries."""
    if n * 3 % 2:
        raise ValueError("3-regular graphs need an even vertex count")
    while True:
        stubs = [v for v in range(n) for _ in range(3)]
        rng.shuffle(stubs)
        edges = set()
        ok = True
        for i in range(0, len(stubs), 2):
            a, b = stubs[i], stubs[i + 1]
            if a == b or (min(a, b), max(a, b)) in edges:
                ok = False
                break
            edges.add((min(a, b), max(a, b)))
        if ok:
            return sorted(edges)


def qaoa_graph(n: int, rng: random.Random) -> list[tuple[int, int]]:
    """c3's MaxCut graph: a seeded 3-regular graph on n vertices. For odd n,
    where no 3-regular graph exists (weak-scaled c3 at 31 / 33 qubits), a
    seeded 3-regular graph on n + 1 vertices with vertex n removed (its three
    neighbours keep degree 2)."""
    if n % 2 == 0:
        return random_3_regular(n, rng)
    return [(a, b) for a, b in random_3_regular(n + 1, rng) if b != n]


def qaoa_config(n: int = 30, layers: int = 4, seed: int = 0) -> Circuit:
    """c3: H on all; per layer ZZ(gamma) on every edge of a seeded
    3-regular graph (``qaoa_graph``) as CX, RZ(2 gamma), CX (bench.qaoa
    convention), then RX(2 beta) on every qubit; gamma, beta ~ U[0, pi)."""
    rng = random.Random(seed)
    edges = qaoa_graph(n, rng)
    angles = [(rng.uniform(0, _PI), rng.uniform(0, _PI)) for _ in range(layers)]
    ops = [_op(GateKind.H, q) for q in range(n)]
    for gamma, beta in angles:
        for u, v in edges:
            ops += [_op(GateKind.CX, u, v), _op(GateKind.RZ, v, params=(2 * gamma,)), _op(GateKind.CX, u, v)]
        ops += [_op(GateKind.RX, q, params=(2 * beta,)) for q in range(n)]
    return Circuit(n, tuple(ops))


def ising_config(n: int = 33, steps: int = 50, seed: int = 0, dt: float = 0.1) -> Circuit:
    """c4: open-chain TFIM Trotter steps: RZZ(i, i+1; J dt) as CX.RZ.CX for
    every bond, then RX(q; h dt); J, h ~ U[0.5, 1.5] seeded."""
    rng = random.Random(seed)
    J = rng.uniform(0.5, 1.5)
    h = rng.uniform(0.5, 1.5)
    ops = []
    for _ in range(steps):
        for i in range(n - 1):
            ops += [_op(GateKind.CX, i, i + 1), _op(GateKind.RZ, i + 1, params=(J * dt,)), _op(GateKind.CX, i, i + 1)]
        ops += [_op(GateKind.RX, q, params=(h * dt,)) for q in range(n)]
    return Circuit(n, tuple(ops))


@dataclass(frozen=True)
class Config:
    name: str
    description: str
    num_qubits: int
    limit: int
    gpus: int
    seed: int = 0

    def circuit(self) -> Circuit:
        return build(self.name, self.seed)


CONFIGS = {
    "c1": Config("c1", "20-qubit QFT (seeded X prefix), complex128, k=10", 20, 10, 1),
    "c2": Config("c2", "26-qubit random supremacy-style, 5x5+1 grid, depth 20, complex128, k=12", 26, 12, 1),
    "c3": Config("c3", "30-qubit QAOA MaxCut p=4 on a seeded 3-regular graph, complex128, k=12", 30, 12, 1),
    "c4": Config("c4", "33-qubit TFIM Trotter chain, 50 steps, complex128, k=12, 2/4/8 GPUs", 33, 12, 8),
    "c5": Config("c5", "36-qubit random circuit, 6x6 grid, depth 24, complex128, k=14, 8 GPUs", 36, 14, 8),
    "c5_35": Config("c5_35", "35-qubit random circuit (6x6 minus corner (5,5)), depth 24, 4 GPUs", 35, 14, 4),
    "c5_34": Config("c5_34", "34-qubit random circuit (6x6 minus corners (5,5),(0,5)), depth 24, 2 GPUs", 34, 14, 2),
    # one GPU's share of c5: 33 local qubits (128 GiB), the same k = 14 parts
    "c5_33": Config("c5_33", "33-qubit random circuit (6x6 minus corners (5,5),(0,5),(5,0)), depth 24, k=14: "
                    "the per-GPU state size of c5 on 8 GPUs", 33, 14, 1),
}


def build(name: str, seed: int = 0) -> Circuit:
    """Circuit of a named config (or a scaled variant like ``c2@20``:
    the same generator at 20 qubits, for tests)."""
    base, _, size = name.partition("@")
    if base == "c1":
        return qft_config(int(size) if size else 20, seed)
    if base == "c2":
        if size:
            n = int(size)
            cols, sites = 5, n - 1
            rows = -(-sites // cols)
            return random_grid_circuit(rows, cols, 20, seed, drop=_fix_drop(rows, cols, sites),
                                       extra_at=(rows // 2, cols // 2))
        return random_grid_circuit(5, 5, 20, seed, extra_at=(2, 2))
    if base == "c3":
        return qaoa_config(int(size) if size else 30, 4, seed)
    if base == "c4":
        return ising_config(int(size) if size else 33, 50, seed)
    if base.startswith("c5"):
        # c5 (36 q on 8 GPUs) and its weak-scaling members: 6x6 grid minus
        # corners (5,5), (0,5), (5,0) for 35 / 34 / 33 qubits
        sizes = {"c5": 36, "c5_35": 35, "c5_34": 34, "c5_33": 33}
        if base not in sizes:
            raise KeyError(f"unknown config {name!r}")
        n = int(size) if size else sizes[base]
        if size and base != "c5":
            raise KeyError(f"{base} has a fixed size; use c5@{n}")
        corners = ((5, 5), (0, 5), (5, 0))
        if not 33 <= n <= 36:
            raise KeyError(f"c5 is defined for 33..36 qubits, not {n}")
        return random_grid_circuit(6, 6, 24, seed, drop=corners[:36 - n])
    raise KeyError(f"unknown config {name!r}")


#: what ``bench.py --config X --gpus N`` runs: (circuit name, scaling).
#: c1 / c2 / c3 weak-scale (n + log2 N qubits: a fixed 2^n shard per GPU);
#: c4 is BASELINE's strong-scaling case (33 qubits over 2 / 4 / 8 GPUs; one
#: GPU holds all 128 GiB in place); c5 is 36 qubits on 8 GPUs with BASELINE's
#: weak-scaling members 35 / 4, 34 / 2 and their one-GPU share 33 / 1.
C5_BY_GPUS = {1: "c5_33", 2: "c5_34", 4: "c5_35", 8: "c5"}


def bench_workload(config: str, gpus: int) -> tuple[str, str]:
    if gpus < 1 or gpus & (gpus - 1):
        raise ValueError(f"--gpus must be a power of two, not {gpus}")
    extra = gpus.bit_length() - 1
    base, _, size = config.partition("@")
    if base not in CONFIGS:
        raise KeyError(f"unknown config {config!r}")
    if base == "c4":
        return (config, "strong")
    if base.startswith("c5"):
        if base == "c5" and not size:
            if gpus not in C5_BY_GPUS:
                raise ValueError(f"c5 runs on 1, 2, 4 or 8 GPUs, not {gpus}")
            return (C5_BY_GPUS[gpus], "weak")
        if gpus != 1:
            raise ValueError(f"{config} is one member of c5's weak-scaling family; run --config c5 --gpus {gpus}")
        return (config, "weak")
    n = int(size) if size else CONFIGS[base].num_qubits
    return ((f"{base}@{n + extra}" if extra else config), "weak")


def _fix_drop(rows: int, cols: int, sites: int):
    """Drop trailing sites of the last grid row so the grid holds ``sites``."""
    surplus = rows * cols - sites
    return tuple((rows - 1, cols - 1 - i) for i in range(surplus))
