"""Acyclic partitioning of the gate DAG under a working-set limit (host).

Produces exactly the partitions of the reference partitioners
(/root/reference/pkg/src/hisim/partition.py) so part order and qubit sets
match ("identical part order and qubit maps", BASELINE.json north_star):

* ``partition_nat``   ~ partition.py:224-228 (cutoff scan, program order)
* ``partition_dfs``   ~ partition.py:231-253 (cutoff scan, best of seeded DFS
  orders)
* ``partition_dagp``  ~ partition.py:258-393 (recursive prefix bisection with
  boundary refinement, then greedy merge, then Kahn relabel)
* ``partition_multilevel`` ~ partition.py:628-678

The dagP merge phase keeps the reference's heap discipline (same keys, same
lazy revalidation, hence the same merge sequence) but maintains the part
graph incrementally and prunes the acyclicity DFS with a topological
potential, instead of rebuilding adjacency and running an unbounded DFS for
every candidate (where the reference spends >40 min
on config 4). Both give the same booleans, so the output is identical.
"""

from __future__ import annotations

import heapq
import json
import math
from dataclasses import dataclass

from .dag import GateDag, NodeKind, build_dag, dfs_topo_order, quotient_is_acyclic
from .errors import LimitTooSmallError, PartitionError
from .qasm import Circuit, GateOp

#: bisection balance window: a side holds at most eps * half the segment
BISECT_EPS = 1.5


@dataclass(frozen=True)
class Part:
    """Gate op indices (ascending program order) and their qubits (ascending)."""

    id: int
    gate_indices: tuple[int, ...]
    qubits: tuple[int, ...]

    @property
    def working_set(self) -> int:
        return len(self.qubits)


@dataclass(frozen=True)
class PartitionResult:
    """A partition whose ``parts`` are in execution (topological) order."""

    strategy: str
    limit: int
    parts: tuple[Part, ...]

    @property
    def num_parts(self) -> int:
        return len(self.parts)

    def part_of(self) -> dict[int, int]:
        """op index -> position of its part in ``parts``."""
        return {g: pos for pos, p in enumerate(self.parts) for g in p.gate_indices}

    def assignment(self, dag: GateDag) -> dict[int, int]:
        """Part of every DAG node; entry stubs follow the first gate on their
        qubit, exit stubs the last, idle qubits go to part 0."""
        where = self.part_of()
        first: dict[int, int] = {}
        last: dict[int, int] = {}
        for i, op in enumerate(dag.circuit.ops):
            for q in op.qubits:
                first.setdefault(q, where[i])
                last[q] = where[i]
        out = {dag.gate_id(i): where[i] for i in range(dag.num_gates)}
        for q in range(dag.num_qubits):
            out[dag.entry_id(q)] = first.get(q, 0)
            out[dag.exit_id(q)] = last.get(q, 0)
        return out

    def _gate_edges(self, dag: GateDag):
        for e in dag.edges:
            a, b = dag.nodes[e.src], dag.nodes[e.dst]
            if a.kind is NodeKind.GATE and b.kind is NodeKind.GATE:
                yield a.op_index, b.op_index

    def part_graph_edges(self, dag: GateDag) -> tuple[tuple[int, int], ...]:
        where = self.part_of()
        return tuple(sorted({(where[a], where[b]) for a, b in self._gate_edges(dag)
                             if where[a] != where[b]}))

    def cut_edges(self, dag: GateDag) -> int:
        where = self.part_of()
        return sum(1 for a, b in self._gate_edges(dag) if where[a] != where[b])


@dataclass(frozen=True)
class MultiLevelPartition:
    """Level-1 partition plus, per level-1 part, a level-2 partition of its
    gates and the padded qubit set each level-2 part is staged on."""

    limit1: int
    limit2: int
    level1: PartitionResult
    sublevels: tuple[PartitionResult, ...]
    padded_qubits: tuple[tuple[tuple[int, ...], ...], ...]


# --- helpers ----------------------------------------------------------------

def _require_limit(circuit: Circuit, limit: int) -> None:
    widest = max((len(op.qubits) for op in circuit.ops), default=1)
    if limit < widest:
        raise LimitTooSmallError(limit, widest)


def _gate_succ_pred(dag: GateDag) -> tuple[list[set[int]], list[set[int]]]:
    """Direct gate->gate dependencies by op index (sets, duplicates folded)."""
    m = dag.num_gates
    succ: list[set[int]] = [set() for _ in range(m)]
    pred: list[set[int]] = [set() for _ in range(m)]
    nodes = dag.nodes
    for e in dag.edges:
        a, b = nodes[e.src], nodes[e.dst]
        if a.kind is NodeKind.GATE and b.kind is NodeKind.GATE:
            succ[a.op_index].add(b.op_index)
            pred[b.op_index].add(a.op_index)
    return succ, pred


def _freeze(circuit: Circuit, strategy: str, limit: int, groups) -> PartitionResult:
    parts = []
    for pid, gates in enumerate(groups):
        gates = sorted(gates)
        qs = sorted({q for g in gates for q in circuit.ops[g].qubits})
        parts.append(Part(pid, tuple(gates), tuple(qs)))
    return PartitionResult(strategy, limit, tuple(parts))


def check_partition(dag: GateDag, result: PartitionResult) -> None:
    """Raise ``PartitionError`` unless parts are nonempty, disjoint,
    exhaustive, within the limit, with fresh qubit sets, listed in
    topological order, and the quotient graph is acyclic
    (reference: partition.py:165-199)."""
    ops = dag.circuit.ops
    covered: set[int] = set()
    for p in result.parts:
        if not p.gate_indices:
            raise PartitionError(f"part {p.id} is empty")
        if p.working_set > result.limit:
            raise PartitionError(
                f"part {p.id} needs {p.working_set} qubits, limit {result.limit}"
            )
        if list(p.qubits) != sorted({q for g in p.gate_indices for q in ops[g].qubits}):
            raise PartitionError(f"part {p.id} qubit set is stale")
        dup = covered.intersection(p.gate_indices)
        if dup:
            raise PartitionError(f"gates {sorted(dup)} in two parts")
        covered.update(p.gate_indices)
    missing = set(range(dag.num_gates)) - covered
    if missing:
        raise PartitionError(f"gates {sorted(missing)} unassigned")
    if not result.parts:
        return
    where = result.part_of()
    succ, _ = _gate_succ_pred(dag)
    for a in range(dag.num_gates):
        for b in succ[a]:
            if where[a] > where[b]:
                raise PartitionError(f"parts not topologically ordered: gate {a} -> {b}")
    if not quotient_is_acyclic(dag, result.assignment(dag)):
        raise PartitionError("quotient graph has a cycle")


# --- cutoff scans -----------------------------------------------------------

def _cutoff(circuit: Circuit, order, limit: int) -> list[list[int]]:
    """Grow the current group until the next gate would exceed ``limit``."""
    groups: list[list[int]] = []
    cur: list[int] = []
    cur_q: set[int] = set()
    ops = circuit.ops
    for g in order:
        gq = ops[g].qubits
        grown = cur_q.union(gq)
        if cur and len(grown) > limit:
            groups.append(cur)
            cur, cur_q = [g], set(gq)
        else:
            cur.append(g)
            cur_q = grown
    if cur:
        groups.append(cur)
    return groups


def partition_nat(dag: GateDag, limit: int) -> PartitionResult:
    """Cutoff scan over program order."""
    _require_limit(dag.circuit, limit)
    return _freeze(dag.circuit, "nat", limit, _cutoff(dag.circuit, range(dag.num_gates), limit))


def partition_dfs(dag: GateDag, limit: int, trials: int = 16, seed: int = 0) -> PartitionResult:
    """Cutoff scan over ``trials`` seeded DFS orders (seed + i); fewest parts
    wins, ties to the earliest trial."""
    _require_limit(dag.circuit, limit)
    if trials < 1:
        raise ValueError("trials must be positive")
    nq = dag.num_qubits
    m = dag.num_gates
    best = None
    for t in range(trials):
        order = [nid - nq for nid in dfs_topo_order(dag, seed + t) if nq <= nid < nq + m]
        groups = _cutoff(dag.circuit, order, limit)
        if best is None or len(groups) < len(best):
            best = groups
    return _freeze(dag.circuit, "dfs", limit, best or [])


# --- dagP -------------------------------------------------------------------

class _Bisector:
    """Recursive prefix bisection + single-gate boundary refinement."""

    def __init__(self, qubits_of, succ, pred):
        self.qubits_of = qubits_of
        self.succ = succ
        self.pred = pred

    def run(self, seg: list[int]) -> list[list[int]]:
        out: list[list[int]] = []
        todo = [seg]
        while todo:  # explicit stack, left half first (same order as recursion)
            s = todo.pop()
            if len(s) == 1:
                out.append(s)
                continue
            a, b = self.split(s)
            todo.append(b)
            todo.append(a)
        return out

    def split(self, seg: list[int]) -> tuple[list[int], list[int]]:
        qof = self.qubits_of
        n = len(seg)
        hi = min(n - 1, math.floor(BISECT_EPS * n / 2))
        lo = max(1, n - hi)
        right: dict[int, int] = {}
        for g in seg:
            for q in qof[g]:
                right[q] = right.get(q, 0) + 1
        left: dict[int, int] = {}
        shared = 0
        best_k = best_cost = None
        for k in range(1, hi + 1):
            for q in qof[seg[k - 1]]:
                right[q] -= 1
                before = left.get(q, 0)
                left[q] = before + 1
                if before == 0 and right[q] > 0:
                    shared += 1
                elif before > 0 and right[q] == 0:
                    shared -= 1
            if k < lo:
                continue
            if (best_cost is None or shared < best_cost
                    or (shared == best_cost and abs(k - n / 2) < abs(best_k - n / 2))):
                best_k, best_cost = k, shared
        return self.refine(seg[:best_k], seg[best_k:], lo)

    def refine(self, a: list[int], b: list[int], lo: int):
        qof, succ, pred = self.qubits_of, self.succ, self.pred
        side_a, side_b = set(a), set(b)
        cnt_a: dict[int, int] = {}
        cnt_b: dict[int, int] = {}
        for g in a:
            for q in qof[g]:
                cnt_a[q] = cnt_a.get(q, 0) + 1
        for g in b:
            for q in qof[g]:
                cnt_b[q] = cnt_b.get(q, 0) + 1

        def delta(g, src, dst):
            d = 0
            for q in qof[g]:
                s, t = src[q], dst.get(q, 0)
                d += (1 if s - 1 > 0 and t + 1 > 0 else 0) - (1 if s > 0 and t > 0 else 0)
            return d

        while True:
            pick = None  # (gain, gate, a_to_b)
            if len(side_a) > lo:
                for g in side_a:
                    if succ[g] & side_a:
                        continue
                    d = delta(g, cnt_a, cnt_b)
                    if d < 0 and (pick is None or d < pick[0]):
                        pick = (d, g, True)
            if len(side_b) > lo:
                for g in side_b:
                    if pred[g] & side_b:
                        continue
                    d = delta(g, cnt_b, cnt_a)
                    if d < 0 and (pick is None or d < pick[0]):
                        pick = (d, g, False)
            if pick is None:
                return sorted(side_a), sorted(side_b)
            _, g, a_to_b = pick
            if a_to_b:
                side_a.remove(g)
                side_b.add(g)
                src, dst = cnt_a, cnt_b
            else:
                side_b.remove(g)
                side_a.add(g)
                src, dst = cnt_b, cnt_a
            for q in qof[g]:
                src[q] -= 1
                dst[q] = dst.get(q, 0) + 1


class _PartGraph:
    """Part-level DAG with incremental contraction and a topological
    potential ``pot`` (pot[a] < pot[b] for every edge a->b) that bounds the
    reachability search."""

    def __init__(self, groups, succ):
        part_of = {}
        for i, gs in enumerate(groups):
            for g in gs:
                part_of[g] = i
        self.out = {i: set() for i in range(len(groups))}
        self.inn = {i: set() for i in range(len(groups))}
        for g, ss in enumerate(succ):
            for s in ss:
                a, b = part_of[g], part_of[s]
                if a != b:
                    self.out[a].add(b)
                    self.inn[b].add(a)
        self.pot = {}
        indeg = {p: len(self.inn[p]) for p in self.out}
        ready = [p for p in self.out if indeg[p] == 0]
        level = dict.fromkeys(self.out, 0)
        while ready:
            p = ready.pop()
            for b in self.out[p]:
                if level[p] + 1 > level[b]:
                    level[b] = level[p] + 1
                indeg[b] -= 1
                if indeg[b] == 0:
                    ready.append(b)
        self.pot = level

    def reaches_indirectly(self, src: int, dst: int) -> bool:
        """Is there a path src -> ... -> dst other than the edge src->dst?"""
        pot, out = self.pot, self.out
        limit = pot[dst]
        stack = []
        seen = set()
        for m in out[src]:
            if m != dst and pot[m] < limit:
                stack.append(m)
                seen.add(m)
        while stack:
            x = stack.pop()
            for y in out[x]:
                if y == dst:
                    return True
                if y not in seen and pot[y] < limit:
                    seen.add(y)
                    stack.append(y)
        return False

    def contract(self, u: int, v: int) -> None:
        """Merge v into u (caller guarantees the result stays acyclic)."""
        out, inn, pot = self.out, self.inn, self.pot
        for b in out.pop(v):
            inn[b].discard(v)
            if b != u:
                out[u].add(b)
                inn[b].add(u)
        for a in inn.pop(v):
            out[a].discard(v)
            if a != u:
                inn[u].add(a)
                out[a].add(u)
        out[u].discard(u)
        inn[u].discard(u)
        # restore the potential: u must sit above all its predecessors
        p = max(pot.pop(v), pot[u])
        for a in inn[u]:
            if pot[a] + 1 > p:
                p = pot[a] + 1
        pot[u] = p
        stack = [u]
        while stack:
            x = stack.pop()
            for b in out[x]:
                if pot[b] <= pot[x]:
                    pot[b] = pot[x] + 1
                    stack.append(b)


def _merge_groups(groups, qubits_of, succ, limit):
    """The merge phase: the host C++ restatement (hs_dagp_merge) when the
    circuit fits 64-qubit masks and the library loads, else Python."""
    if _NATIVE_MERGE:
        merged = _merge_groups_native(groups, qubits_of, succ, limit)
        if merged is not None:
            return merged
    return _merge_groups_py(groups, qubits_of, succ, limit)


#: use hs_dagp_merge (tests flip this to compare with the Python merge)
_NATIVE_MERGE = True


def _merge_groups_native(groups, qubits_of, succ, limit):
    import ctypes

    try:
        from . import _native

        lib = _native.load()
    except Exception:  # no library on this host: the Python merge
        return None
    G = len(groups)
    masks = (ctypes.c_uint64 * max(1, G))()
    where = {}
    for i, gs in enumerate(groups):
        m = 0
        for g in gs:
            where[g] = i
            for q in qubits_of[g]:
                if q >= 64:
                    return None
                m |= 1 << q
        masks[i] = m
    edges = sorted({(where[g], where[s]) for g, ss in enumerate(succ) for s in ss if where[g] != where[s]})
    src = (ctypes.c_int32 * max(1, len(edges)))(*[a for a, _ in edges])
    dst = (ctypes.c_int32 * max(1, len(edges)))(*[b for _, b in edges])
    into = (ctypes.c_int32 * max(1, G))()
    _native.check(lib.hs_dagp_merge(G, masks, len(edges), src, dst, limit, into))
    alive = {}
    for i in range(G):
        alive.setdefault(int(into[i]), set()).update(groups[i])
    return [sorted(alive[p]) for p in sorted(alive)]


def _merge_groups_py(groups, qubits_of, succ, limit):
    """Greedy pair contraction (reference: partition.py:396-478): pop pairs by
    (-shared qubits, -union size, u, v); a popped key is recomputed and
    requeued if stale; a valid pair merges when contraction stays acyclic,
    after which the merged part's pairings are pushed again."""
    alive = {i: set(g) for i, g in enumerate(groups)}
    qset = {i: set().union(*(qubits_of[g] for g in groups[i])) for i in alive}
    graph = _PartGraph(groups, succ)

    def key(u, v):
        qu, qv = qset[u], qset[v]
        union = len(qu | qv)
        if union > limit:
            return None
        return (union - len(qu) - len(qv), -union, u, v)  # (-shared, -union, u, v)

    ids = sorted(alive)
    heap = []
    for i, u in enumerate(ids):
        for v in ids[i + 1:]:
            k = key(u, v)
            if k is not None:
                heap.append(k)
    heapq.heapify(heap)
    pop, push = heapq.heappop, heapq.heappush
    while heap:
        entry = pop(heap)
        u, v = entry[2], entry[3]
        if u not in alive or v not in alive:
            continue
        k = key(u, v)
        if k is None:
            continue
        if k != entry:
            push(heap, k)
            continue
        if graph.reaches_indirectly(u, v) or graph.reaches_indirectly(v, u):
            continue
        alive[u] |= alive.pop(v)
        qset[u] |= qset.pop(v)
        graph.contract(u, v)
        for w in alive:
            if w != u:
                k = key(u, w) if u < w else key(w, u)
                if k is not None:
                    push(heap, k)
    return [sorted(alive[p]) for p in sorted(alive)]


def _kahn_relabel(groups, succ):
    """Order groups topologically, smallest group index first."""
    where = {g: i for i, gs in enumerate(groups) for g in gs}
    out = [set() for _ in groups]
    indeg = [0] * len(groups)
    for g, ss in enumerate(succ):
        for s in ss:
            a, b = where[g], where[s]
            if a != b and b not in out[a]:
                out[a].add(b)
                indeg[b] += 1
    ready = [i for i in range(len(groups)) if indeg[i] == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        a = heapq.heappop(ready)
        order.append(groups[a])
        for b in out[a]:
            indeg[b] -= 1
            if indeg[b] == 0:
                heapq.heappush(ready, b)
    if len(order) != len(groups):
        raise PartitionError("internal: merged part graph is cyclic")
    return order


def partition_dagp(dag: GateDag, limit: int) -> PartitionResult:
    """dagP-style partition: bisect to single gates, refine boundaries,
    greedily merge under the limit keeping the part graph acyclic, then
    relabel topologically."""
    circuit = dag.circuit
    _require_limit(circuit, limit)
    m = dag.num_gates
    if m == 0:
        return PartitionResult("dagp", limit, ())
    succ, pred = _gate_succ_pred(dag)
    qubits_of = [set(op.qubits) for op in circuit.ops]
    if len(set().union(*qubits_of)) <= limit:
        return _freeze(circuit, "dagp", limit, [list(range(m))])
    groups = _Bisector(qubits_of, succ, pred).run(list(range(m)))
    groups = _merge_groups(groups, qubits_of, succ, limit)
    return _freeze(circuit, "dagp", limit, _kahn_relabel(groups, succ))


# --- two levels -------------------------------------------------------------

def partition_multilevel(dag: GateDag, limit1: int, limit2: int) -> MultiLevelPartition:
    """dagP at ``limit1``, then dagP of each part's own sub-circuit at
    ``min(limit2, w)``; level-2 parts are padded with parent qubits (lowest
    first) up to that width (reference: partition.py:628-678)."""
    if limit2 > limit1:
        raise PartitionError(f"limit2 {limit2} exceeds limit1 {limit1}")
    level1 = partition_dagp(dag, limit1)
    subs, pads = [], []
    ops = dag.circuit.ops
    for part in level1.parts:
        local = {q: s for s, q in enumerate(part.qubits)}
        sub_circuit = Circuit(
            len(part.qubits),
            tuple(GateOp(ops[g].kind, tuple(local[q] for q in ops[g].qubits), ops[g].params)
                  for g in part.gate_indices),
        )
        width = min(limit2, len(part.qubits))
        inner = partition_dagp(build_dag(sub_circuit), width)
        mapped, padded = [], []
        for sp in inner.parts:
            qs = tuple(sorted(part.qubits[s] for s in sp.qubits))
            mapped.append(Part(sp.id, tuple(sorted(part.gate_indices[i] for i in sp.gate_indices)), qs))
            pad = list(qs)
            for q in part.qubits:
                if len(pad) >= width:
                    break
                if q not in qs:
                    pad.append(q)
            padded.append(tuple(sorted(pad)))
        subs.append(PartitionResult("dagp", limit2, tuple(mapped)))
        pads.append(tuple(padded))
    return MultiLevelPartition(limit1, limit2, level1, tuple(subs), tuple(pads))


# --- JSON -------------------------------------------------------------------

def _part_doc(p: Part) -> dict:
    return {"id": p.id, "gate_indices": list(p.gate_indices),
            "qubits": list(p.qubits), "working_set": p.working_set}


def partition_to_json(dag: GateDag, result: PartitionResult) -> str:
    """Same document as the reference (partition.py:683-701)."""
    return json.dumps({
        "strategy": result.strategy,
        "limit": result.limit,
        "num_parts": result.num_parts,
        "parts": [_part_doc(p) for p in result.parts],
        "edges": [list(e) for e in result.part_graph_edges(dag)],
        "cut_edges": result.cut_edges(dag),
    }, indent=2)


def partition_from_json(dag: GateDag, text: str) -> PartitionResult:
    """Load and validate a ``partition_to_json`` document."""
    doc = json.loads(text)
    result = PartitionResult(
        doc["strategy"], int(doc["limit"]),
        tuple(Part(p["id"], tuple(p["gate_indices"]), tuple(p["qubits"])) for p in doc["parts"]),
    )
    check_partition(dag, result)
    return result


def multilevel_to_json(dag: GateDag, ml: MultiLevelPartition) -> str:
    return json.dumps({
        "strategy": "multilevel",
        "limit1": ml.limit1,
        "limit2": ml.limit2,
        "level1": json.loads(partition_to_json(dag, ml.level1)),
        "sublevels": [
            {"parent": ml.level1.parts[i].id,
             "parts": [_part_doc(p) for p in sub.parts],
             "padded_qubits": [list(q) for q in ml.padded_qubits[i]]}
            for i, sub in enumerate(ml.sublevels)
        ],
    }, indent=2)
