"""Host-side parity with the reference: IR, DAG, partitioners, layouts,
communication accounting and trace schemas (no GPU needed)."""

import json
import math
import random

import numpy as np
import pytest

from conftest import parts_of, partition_of
from paper_2205_06973_b200 import configs
from paper_2205_06973_b200.dag import build_dag, dfs_topo_order, quotient_is_acyclic, working_set
from paper_2205_06973_b200.dist import (
    RankLayout,
    choose_layout,
    default_layout,
    plan_layouts,
    plan_redistribution,
    switch_stats,
)
from paper_2205_06973_b200.errors import (
    DuplicateQubitError,
    InvalidQubitCountError,
    LayoutMismatchError,
    LimitTooSmallError,
    PartitionError,
    PartTooWideForLayoutError,
    QasmSyntaxError,
    QubitOutOfRangeError,
    UnsupportedGateError,
)
from paper_2205_06973_b200.hier import QubitSlotMap, bit_offsets, gather, part_block_indices, remap_part, scatter
from paper_2205_06973_b200.partition import (
    Part,
    check_partition,
    partition_dagp,
    partition_dfs,
    partition_from_json,
    partition_multilevel,
    partition_nat,
    partition_to_json,
)
from paper_2205_06973_b200.qasm import Circuit, GateKind, GateOp, parse_qasm, to_qasm

FNS = {"nat": partition_nat, "dfs": partition_dfs, "dagp": partition_dagp}


def test_qasm_round_trip_matches_reference_text(golden):
    for doc in golden.json("corpus"):
        c = parse_qasm(doc["qasm"])
        assert to_qasm(c) == doc["qasm"]
        assert parse_qasm(to_qasm(c)) == c
    for doc in golden.json("bundled").values():
        assert to_qasm(parse_qasm(doc["qasm"])) == doc["qasm"]


def test_qasm_errors():
    with pytest.raises(QasmSyntaxError):
        parse_qasm("OPENQASM 2.0;\nh q[0];")
    with pytest.raises(UnsupportedGateError):
        parse_qasm("qreg q[2];\nmeasure q[0];")
    with pytest.raises(UnsupportedGateError):
        parse_qasm("qreg q[2];\nfoo q[0];")
    with pytest.raises(QubitOutOfRangeError):
        parse_qasm("qreg q[2];\nh q[2];")
    with pytest.raises(DuplicateQubitError):
        parse_qasm("qreg q[2];\ncx q[1],q[1];")
    with pytest.raises(InvalidQubitCountError):
        parse_qasm("qreg q[2];\nrx q[0];")
    with pytest.raises(QasmSyntaxError):
        parse_qasm("qreg q[2];\nrx(pi/0) q[0];")
    c = parse_qasm("qreg q[1];\nrx(-3*pi/4 + 2^2) q[0]; // c\nbarrier q[0];")
    assert math.isclose(c.ops[0].params[0], -3 * math.pi / 4 + 4)


def test_dag_shape_and_working_set():
    c = configs.build("c1@6")
    d = build_dag(c)
    assert len(d.nodes) == c.num_ops + 2 * c.num_qubits
    assert len(d.edges) == c.num_qubits + sum(len(op.qubits) for op in c.ops)
    assert working_set(d, [d.gate_id(i) for i in range(c.num_ops)]) == c.num_qubits
    order = dfs_topo_order(d, 3)
    pos = {nid: i for i, nid in enumerate(order)}
    assert all(pos[e.src] < pos[e.dst] for e in d.edges)
    assert dfs_topo_order(d, 3) == order


def test_partitions_match_reference_on_corpus(golden):
    for doc in golden.json("corpus"):
        c = parse_qasm(doc["qasm"])
        d = build_dag(c)
        for key, want in doc["partitions"].items():
            name, lim = key.split("@")
            got = FNS[name](d, int(lim))
            assert [[list(p.gate_indices), list(p.qubits)] for p in got.parts] == want, key
            check_partition(d, got)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5", "c4@small"])
def test_partitions_match_reference_on_configs(golden, name):
    doc = golden.json("configs")[name]
    c = configs.ising_config(33, 5) if name == "c4@small" else configs.build(name)
    assert (c.num_qubits, c.num_ops) == (doc["num_qubits"], doc["num_ops"])
    d = build_dag(c)
    for strategy, want in doc["partitions"].items():
        got = FNS[strategy](d, doc["limit"])
        assert [[list(p.gate_indices), list(p.qubits)] for p in got.parts] == want, strategy


def test_multilevel_partitions_and_trace_rows(golden):
    from paper_2205_06973_b200.hier import multilevel_trace

    for name, doc in golden.json("bundled").items():
        if "multilevel" not in doc:
            continue
        c = parse_qasm(doc["qasm"])
        ml = doc["multilevel"]
        got = partition_multilevel(build_dag(c), ml["limit1"], ml["limit2"])
        assert [[list(p.gate_indices), list(p.qubits)] for p in got.level1.parts] == ml["level1"]
        assert [[[list(p.gate_indices), list(p.qubits)] for p in s.parts] for s in got.sublevels] == ml["sublevels"]
        assert [[list(q) for q in pads] for pads in got.padded_qubits] == ml["padded"]
        assert multilevel_trace(c, got).part_rows() == ml["trace"]


def test_nat_trace_rows_match_reference(golden):
    from paper_2205_06973_b200.hier import hierarchical_trace

    for name, doc in golden.json("bundled").items():
        c = parse_qasm(doc["qasm"])
        part = partition_nat(build_dag(c), doc["limit"])
        assert hierarchical_trace(c, part).part_rows() == doc["nat_trace"]


def test_partition_json_round_trip_and_validation():
    c = configs.build("c2@12")
    d = build_dag(c)
    res = partition_dagp(d, 6)
    back = partition_from_json(d, partition_to_json(d, res))
    assert back == res
    bad = json.loads(partition_to_json(d, res))
    bad["parts"][0]["qubits"] = bad["parts"][0]["qubits"][:-1]
    with pytest.raises(PartitionError):
        partition_from_json(d, json.dumps(bad))
    with pytest.raises(LimitTooSmallError):
        partition_nat(build_dag(Circuit(3, (GateOp(GateKind.CCX, (0, 1, 2)),))), 2)


def test_addressing_helpers(golden):
    kat = golden.json("kat")
    for bits, expect in kat["bit_offsets"]:
        assert bit_offsets(bits).tolist() == expect
    for n, qubits, a, expect in kat["gather"]:
        data = np.arange(1 << n, dtype=np.complex128)
        assert gather(data, n, qubits, a).real.astype(int).tolist() == expect
    for n, qubits, expect in kat["block_indices"]:
        assert part_block_indices(n, qubits).tolist() == expect
    data = np.arange(16, dtype=np.complex128)
    inner = gather(data, 4, (1, 2), 2)
    scatter(data, 4, (1, 2), 2, inner * 2)
    assert np.array_equal(data[part_block_indices(4, (1, 2))[2]], inner * 2)
    with pytest.raises(ValueError):
        QubitSlotMap((3, 1))
    m = QubitSlotMap((2, 5, 7))
    assert (m.slot_of(5), m.global_of(2)) == (1, 7)


def test_remap_part_slots():
    c = Circuit(6, (GateOp(GateKind.CX, (4, 1)), GateOp(GateKind.H, (4,))))
    exe = remap_part(c, Part(0, (0, 1), (1, 4)), position_of={1: 3, 4: 0, 2: 5}, stage_qubits=(1, 2, 4))
    assert exe.slot_map.qubits == (0, 3, 5)
    assert exe.op_slots == ((0, 1), (0,))


def test_layouts_match_reference(golden):
    kat = golden.json("kat")
    for n, local, process, g, expect in kat["address_of"]:
        assert list(RankLayout(n, tuple(local), tuple(process)).address_of(g)) == expect
    for n, p, qubits, local, process in kat["choose_layout"]:
        lay = choose_layout(n, p, Part(0, (0,), tuple(qubits)))
        assert (list(lay.local), list(lay.process)) == (local, process)
    assert default_layout(4, 2).process == (2, 3)
    with pytest.raises(PartTooWideForLayoutError):
        choose_layout(4, 3, Part(0, (0,), (0, 1)))
    with pytest.raises(LayoutMismatchError):
        switch_stats(1, RankLayout(4, (0, 1), (2, 3)), RankLayout(5, (0, 1, 2), (3, 4)))


def _stats_dict(s):
    return {"from": s.from_part, "to": s.to_part, "runs": s.num_runs, "messages": s.messages,
            "bytes_remote": s.bytes_remote, "bytes_resident": s.bytes_resident,
            "sent_bytes": {str(k): v for k, v in s.sent_bytes.items()},
            "received_bytes": {str(k): v for k, v in s.received_bytes.items()}}


def test_closed_form_switch_stats_match_reference_plans(golden):
    for n, ol, op, nl, nproc, want in golden.json("kat")["plans"]:
        old = RankLayout(n, tuple(ol), tuple(op))
        new = RankLayout(n, tuple(nl), tuple(nproc))
        assert _stats_dict(switch_stats(1, old, new)) == want
        from paper_2205_06973_b200.dist import SwitchStats

        assert _stats_dict(SwitchStats.from_plan(1, plan_redistribution(old, new))) == want


def test_distributed_layout_policy_matches_reference(golden):
    for doc in golden.json("corpus"):
        c = parse_qasm(doc["qasm"])
        for d in doc["dist"]:
            part = partition_of(d["parts"])
            _, layouts, switches = plan_layouts(c, part, d["p"])
            assert [[list(l.local), list(l.process)] for l in layouts] == d["layouts"]
            assert [_stats_dict(s) for _, _, _, s in switches] == d["switches"]


def test_closed_form_scales_to_36_qubits():
    c = configs.build("c5")
    part = partition_dfs(build_dag(c), 14)
    _, layouts, switches = plan_layouts(c, part, 3)
    assert switches and all(s.bytes_remote + s.bytes_resident == 16 << 36 for *_, s in switches)


@pytest.mark.parametrize("name,limit", [("c1", 10), ("c2@16", 8), ("c3@18", 6), ("c3", 12), ("c2", 12)])
def test_native_dagp_merge_matches_python(name, limit):
    """hs_dagp_merge (C++ restatement of the dagP merge phase) gives the same
    partition as the Python merge, which the corpus goldens pin to the
    reference."""
    import paper_2205_06973_b200.partition as P
    from paper_2205_06973_b200 import build_dag, configs, partition_dagp

    d = build_dag(configs.build(name))
    try:
        P._NATIVE_MERGE = True
        a = partition_dagp(d, limit)
        P._NATIVE_MERGE = False
        b = partition_dagp(d, limit)
    finally:
        P._NATIVE_MERGE = True
    assert [(p.gate_indices, p.qubits) for p in a.parts] == [(p.gate_indices, p.qubits) for p in b.parts]


def test_native_dagp_merge_on_tfim_chain():
    import paper_2205_06973_b200.partition as P
    from paper_2205_06973_b200 import build_dag, partition_dagp
    from paper_2205_06973_b200.configs import ising_config

    d = build_dag(ising_config(20, 6))
    try:
        P._NATIVE_MERGE = False
        b = partition_dagp(d, 8)
    finally:
        P._NATIVE_MERGE = True
    a = partition_dagp(d, 8)
    assert [(p.gate_indices, p.qubits) for p in a.parts] == [(p.gate_indices, p.qubits) for p in b.parts]


@pytest.mark.parametrize("name,limit,p", [("c5", 14, 3), ("c3", 12, 3), ("c4@20", 8, 2), ("c2", 12, 1)])
def test_lookahead_remap_policy(name, limit, p):
    """plan_layouts(policy="lookahead"): every part's qubits are local in its
    layout, consecutive layouts differ only where a part needed a rank
    qubit, and the remote volume never exceeds the reference policy's."""
    from paper_2205_06973_b200 import build_dag, configs, partition_dfs

    c = configs.build(name)
    part = partition_dfs(build_dag(c), limit)
    _, ref_layouts, ref_sw = plan_layouts(c, part, p, "reference")
    first, layouts, sw = plan_layouts(c, part, p, "lookahead")
    for lay, pt in zip(layouts, part.parts):
        assert all(lay.is_local(q) for q in pt.qubits)
    at = {i: (old, new) for i, old, new, _ in sw}
    prev = first
    for i, lay in enumerate(layouts):
        if i in at:
            assert at[i][0] == prev and at[i][1] == lay and lay != prev
        else:
            assert lay == prev
        prev = lay
    assert sum(s.bytes_remote for *_, s in sw) <= sum(s.bytes_remote for *_, s in ref_sw)
    assert len(sw) <= len(ref_sw)
