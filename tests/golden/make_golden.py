"""Generate the golden fixtures from the reference package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the UNMODIFIED reference (``hisim`` from
/root/reference/pkg/src, bytecode writing disabled so nothing is written
there) and records, for inputs built by this repo's generators:

* kat.json      - known answers: bit_offsets, gather, block indices, gate
                  matrices, layout addressing, choose_layout, and full
                  SwitchStats of plan_redistribution for random layout pairs;
* corpus.json / corpus.npz
                - circuits of the reference acceptance corpus generator
                  (CORPUS_SEED 20260822, tests/test_acceptance.py:41-79),
                  their reference partitions (nat/dfs/dagp), flat states,
                  distributed CommStats + layouts at p = 1..3;
* bundled.json / bundled.npz
                - the reference's bundled desk circuits (bench.py) with
                  partitions, multilevel partitions, traces and flat states;
* configs.json / configs.npz
                - reference partitions of the BASELINE configs (c1..c5) and
                  sampled reference amplitudes of scaled configs.

Nothing from these files is needed at run time on the GPU box except the
committed outputs.
"""

from __future__ import annotations

import json
import math
import random
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

import hisim  # noqa: E402  (the reference)
from hisim import bench as rbench  # noqa: E402
from hisim.dag import build_dag as r_build_dag  # noqa: E402
from hisim.dist import (  # noqa: E402
    RankLayout as RLayout,
    choose_layout as r_choose_layout,
    plan_redistribution as r_plan,
    simulate_distributed as r_simdist,
    SwitchStats as RSwitch,
)
from hisim.hier import (  # noqa: E402
    bit_offsets as r_bit_offsets,
    execute_hierarchical as r_exec,
    execute_multilevel as r_exec_ml,
    gather as r_gather,
    part_block_indices as r_pbi,
)
from hisim.partition import (  # noqa: E402
    Part as RPart,
    partition_dagp as r_dagp,
    partition_dfs as r_dfs,
    partition_multilevel as r_ml,
    partition_nat as r_nat,
)
from hisim.qasm import GateKind as RKind, parse_qasm as r_parse, to_qasm as r_to_qasm  # noqa: E402
from hisim.statevec import gate_matrix as r_gate_matrix, simulate_flat as r_flat  # noqa: E402

from paper_2205_06973_b200 import configs as my_configs  # noqa: E402
from paper_2205_06973_b200.qasm import to_qasm as my_to_qasm  # noqa: E402

CORPUS_SEED = 20260822


def cplx(a):
    a = np.asarray(a)
    return [[float(x.real), float(x.imag)] for x in a.reshape(-1)]


def parts_doc(result):
    return [[list(p.gate_indices), list(p.qubits)] for p in result.parts]


def stats_doc(s: RSwitch):
    return {"from": s.from_part, "to": s.to_part, "runs": s.num_runs, "messages": s.messages,
            "bytes_remote": s.bytes_remote, "bytes_resident": s.bytes_resident,
            "sent_bytes": {str(k): v for k, v in s.sent_bytes.items()},
            "received_bytes": {str(k): v for k, v in s.received_bytes.items()}}


def corpus_circuit(rng: random.Random, n: int, num_ops: int):
    """The acceptance corpus generator (test_acceptance.py:56-67)."""
    kinds = list(RKind)
    ops = []
    for _ in range(num_ops):
        kind = rng.choice(kinds)
        if kind.arity > n:
            kind = RKind.CX
        qubits = tuple(rng.sample(range(n), kind.arity))
        params = tuple(rng.uniform(-math.pi, math.pi) for _ in range(kind.num_params))
        ops.append(hisim.GateOp(kind, qubits, params))
    return hisim.Circuit(n, tuple(ops))


def kat():
    doc = {}
    doc["bit_offsets"] = [[b, r_bit_offsets(b).tolist()] for b in ([0, 2], [1], [], [0, 3, 5], [4, 1])]
    doc["gather"] = []
    for n, q, a in [(3, (0,), 0), (2, (1,), 1), (5, (0, 2, 3), 3), (4, (1, 2), 2), (6, (5, 0), 7)]:
        data = np.arange(1 << n, dtype=np.complex128)
        doc["gather"].append([n, list(q), a, r_gather(data, n, q, a).real.astype(int).tolist()])
    doc["block_indices"] = [[n, list(q), r_pbi(n, q).tolist()] for n, q in [(5, (1, 3)), (4, (0, 1, 2, 3)), (6, (0, 4))]]
    rng = random.Random(5)
    doc["gate_matrices"] = []
    for kind in RKind:
        params = tuple(rng.uniform(-2 * math.pi, 2 * math.pi) for _ in range(kind.num_params))
        doc["gate_matrices"].append([kind.value, list(params), cplx(r_gate_matrix(kind, params))])
    lay = RLayout(4, (0, 2), (1, 3))
    doc["address_of"] = [[4, [0, 2], [1, 3], g, list(lay.address_of(g))] for g in range(16)]
    doc["choose_layout"] = []
    for _ in range(60):
        n = rng.randint(2, 10)
        p = rng.randint(0, n - 1)
        w = rng.randint(1, n - p)
        qs = tuple(sorted(rng.sample(range(n), w)))
        lay = r_choose_layout(n, p, RPart(0, (0,), qs))
        doc["choose_layout"].append([n, p, list(qs), list(lay.local), list(lay.process)])
    doc["plans"] = []
    for _ in range(150):
        n = rng.randint(2, 10)
        p = rng.randint(0, min(3, n))
        def rand_layout():
            perm = list(range(n))
            rng.shuffle(perm)
            return RLayout(n, tuple(sorted(perm[: n - p])), tuple(sorted(perm[n - p:])))
        old, new = rand_layout(), rand_layout()
        plan = r_plan(old, new)
        doc["plans"].append([n, list(old.local), list(old.process), list(new.local), list(new.process),
                             stats_doc(RSwitch.from_plan(1, plan))])
    return doc


def corpus(count=60):
    rng = random.Random(CORPUS_SEED)
    docs, states = [], {}
    drng = random.Random(CORPUS_SEED + 7)
    for i in range(count):
        n = rng.randint(3, 12)
        c = corpus_circuit(rng, n, rng.randint(1, 150))
        dag = r_build_dag(c)
        widest = max((len(op.qubits) for op in c.ops), default=1)
        limits = sorted({max(2, widest), max(2, widest, (n + 1) // 2), n})
        entry = {"qasm": r_to_qasm(c), "partitions": {}, "dist": []}
        for lim in limits:
            for name, fn in (("nat", r_nat), ("dfs", r_dfs), ("dagp", r_dagp)):
                entry["partitions"][f"{name}@{lim}"] = parts_doc(fn(dag, lim))
        flat = r_flat(c, max_qubits=n)
        states[f"c{i}"] = flat.data
        # distributed at p = 1..3 with a dagp partition that fits the locals
        for p in (1, 2, 3):
            if n - p < max(2, widest):
                continue
            lim = drng.randint(max(2, widest), n - p)
            part = r_dagp(dag, lim)
            run = r_simdist(c, part, p, max_qubits=n)
            err = float(np.max(np.abs(run.state.data - flat.data)))
            entry["dist"].append({"p": p, "limit": lim, "parts": parts_doc(part),
                                  "switches": [stats_doc(s) for s in run.stats.switches],
                                  "layouts": [[list(l.local), list(l.process)] for l in run.layouts],
                                  "ref_err": err})
        docs.append(entry)
    return docs, states


def bundled():
    docs, states = {}, {}
    for name in rbench.DESK_NAMES:
        c = rbench.build(name)
        n = c.num_qubits
        if n > 14:
            continue
        dag = r_build_dag(c)
        lim = max(2, n // 2)
        e = {"qasm": r_to_qasm(c), "limit": lim, "partitions": {}}
        for pname, fn in (("nat", r_nat), ("dfs", r_dfs), ("dagp", r_dagp)):
            e["partitions"][pname] = parts_doc(fn(dag, lim))
        if n >= 4:
            l1, l2 = max(3, n // 2), max(2, n // 3)
            widest = max(len(op.qubits) for op in c.ops)
            l2 = max(l2, widest)
            l1 = max(l1, l2)
            ml = r_ml(dag, l1, l2)
            state, trace = r_exec_ml(c, ml, with_trace=True, max_qubits=n)
            e["multilevel"] = {"limit1": l1, "limit2": l2, "level1": parts_doc(ml.level1),
                               "sublevels": [parts_doc(s) for s in ml.sublevels],
                               "padded": [[list(q) for q in pads] for pads in ml.padded_qubits],
                               "trace": trace.part_rows()}
        st, tr = r_exec(c, r_nat(dag, lim), with_trace=True, max_qubits=n)
        e["nat_trace"] = tr.part_rows()
        states[name] = r_flat(c, max_qubits=n).data
        docs[name] = e
    return docs, states


def configs():
    doc, arrays = {}, {}
    plan = {
        "c1": (10, ("nat", "dfs", "dagp")),
        "c2": (12, ("nat", "dfs", "dagp")),
        "c3": (12, ("nat", "dfs", "dagp")),
        "c4": (12, ("nat", "dfs")),
        "c5": (14, ("nat", "dfs", "dagp")),
        "c4@small": (12, ("nat", "dfs", "dagp")),
    }
    fns = {"nat": r_nat, "dfs": r_dfs, "dagp": r_dagp}
    for name, (k, strategies) in plan.items():
        mine = my_configs.ising_config(33, 5) if name == "c4@small" else my_configs.build(name)
        text = my_to_qasm(mine)
        c = r_parse(text)  # the reference parses our text: same op list
        assert r_to_qasm(c) == text
        dag = r_build_dag(c)
        entry = {"num_qubits": c.num_qubits, "num_ops": c.num_ops, "limit": k, "partitions": {}, "seconds": {}}
        for s in strategies:
            t0 = time.perf_counter()
            res = fns[s](dag, k)
            entry["seconds"][s] = time.perf_counter() - t0
            entry["partitions"][s] = parts_doc(res)
            print(f"{name} {s}: {res.num_parts} parts ({entry['seconds'][s]:.1f}s)", flush=True)
        doc[name] = entry
    # sampled reference amplitudes of configs small enough for the reference
    srng = np.random.default_rng(2205)
    for name, strategy, k in (("c1", "dagp", 10), ("c2@20", "dfs", 12), ("c3@20", "dfs", 12), ("c4@small18", "dfs", 12)):
        if name == "c4@small18":
            mine = my_configs.ising_config(18, 4)
        else:
            mine = my_configs.build(name)
        c = r_parse(my_to_qasm(mine))
        dag = r_build_dag(c)
        res = fns[strategy](dag, k)
        t0 = time.perf_counter()
        st = r_exec(c, res, max_qubits=c.num_qubits)
        secs = time.perf_counter() - t0
        idx = np.sort(srng.choice(1 << c.num_qubits, size=4096, replace=False))
        key = name.replace("@", "_")
        arrays[key + "_idx"] = idx
        arrays[key + "_amp"] = st.data[idx]
        doc[name + ":sample"] = {"strategy": strategy, "limit": k, "partition": parts_doc(res),
                                 "norm": float(np.linalg.norm(st.data)), "ref_seconds": secs,
                                 "checksum_abs2_weighted": float(np.sum(np.abs(st.data) ** 2 * (np.arange(st.data.size) % 7)))}
        print(f"{name}: reference execute_hierarchical {secs:.1f}s", flush=True)
    return doc, arrays


def main():
    t0 = time.time()
    (HERE / "kat.json").write_text(json.dumps(kat()))
    docs, states = corpus()
    (HERE / "corpus.json").write_text(json.dumps(docs))
    np.savez_compressed(HERE / "corpus.npz", **states)
    docs, states = bundled()
    (HERE / "bundled.json").write_text(json.dumps(docs))
    np.savez_compressed(HERE / "bundled.npz", **states)
    doc, arrays = configs()
    (HERE / "configs.json").write_text(json.dumps(doc))
    np.savez_compressed(HERE / "configs.npz", **arrays)
    print(f"done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
