"""Pin the CPU oracle (oracle/) to the reference's own outputs.

Every expectation here was produced by the unmodified reference package
(tests/golden/make_golden.py); the oracle may only be trusted by the GPU
parity tests because it passes these.
"""

import math

import numpy as np
import pytest

from conftest import parts_of
from oracle import c_oracle
from oracle import hisim_oracle as orc
from paper_2205_06973_b200 import configs
from paper_2205_06973_b200.qasm import GateKind, parse_qasm


def test_known_answers_addressing(golden):
    kat = golden.json("kat")
    for bits, expect in kat["bit_offsets"]:
        assert orc.bit_offsets(bits).tolist() == expect
    for n, qubits, a, expect in kat["gather"]:
        data = np.arange(1 << n, dtype=np.complex128)
        idx = orc.block_indices(n, qubits)[a]
        assert data[idx].real.astype(int).tolist() == expect
    for n, qubits, expect in kat["block_indices"]:
        assert orc.block_indices(n, qubits).tolist() == expect
    # hier.py golden from the reference tests: bits (0,2) -> 0,1,4,5
    assert orc.bit_offsets([0, 2]).tolist() == [0, 1, 4, 5]


def _full_matrix(kind, params):
    """Dense 2^arity matrix from the oracle's 2x2 + control masking, operand
    0 = most significant bit (the reference gate_matrix convention)."""
    nc = orc.CONTROLLED.get(kind, (kind, 0))[1]
    if kind is GateKind.SWAP:
        return np.eye(4)[[0, 2, 1, 3]]
    dim = 1 << (nc + 1)
    m = np.eye(dim, dtype=np.complex128)
    m[dim - 2:, dim - 2:] = orc.base_matrix(kind, params)
    return m


def test_known_answers_gate_matrices(golden):
    for value, params, expect in golden.json("kat")["gate_matrices"]:
        kind = GateKind(value)
        got = _full_matrix(kind, tuple(params))
        want = np.array([complex(a, b) for a, b in expect]).reshape(got.shape)
        np.testing.assert_allclose(got, want, atol=1e-15)


def test_known_answers_layouts(golden):
    kat = golden.json("kat")
    for n, local, process, g, expect in kat["address_of"]:
        assert list(orc.address_of(local, process, g)) == expect
    for n, p, qubits, local, process in kat["choose_layout"]:
        assert orc.choose_layout(n, p, qubits) == (tuple(local), tuple(process))
    for n, ol, op, nl, nproc, st in kat["plans"]:
        got = orc.plan_stats(n, (tuple(ol), tuple(op)), (tuple(nl), tuple(nproc)))
        assert got["runs"] == st["runs"]
        assert got["messages"] == st["messages"]
        assert got["bytes_remote"] == st["bytes_remote"]
        assert got["bytes_resident"] == st["bytes_resident"]
        assert {str(k): v for k, v in got["sent_bytes"].items()} == st["sent_bytes"]
        assert {str(k): v for k, v in got["received_bytes"].items()} == st["received_bytes"]


def test_flat_and_hierarchical_match_reference_corpus(golden):
    docs, states = golden.json("corpus"), golden.npz("corpus")
    worst = 0.0
    for i, doc in enumerate(docs):
        c = parse_qasm(doc["qasm"])
        ref = states[f"c{i}"]
        flat = orc.simulate_flat(c)
        worst = max(worst, float(np.max(np.abs(flat - ref))))
        for key, parts in doc["partitions"].items():
            got = orc.execute_hierarchical(c, parts_of(parts))
            assert np.max(np.abs(got - ref)) < 1e-12, (i, key)
    assert worst < 1e-13


def test_distributed_matches_reference_corpus(golden):
    docs, states = golden.json("corpus"), golden.npz("corpus")
    for i, doc in enumerate(docs):
        c = parse_qasm(doc["qasm"])
        for d in doc["dist"]:
            state, switches, layouts = orc.simulate_distributed(c, parts_of(d["parts"]), d["p"])
            assert np.max(np.abs(state - states[f"c{i}"])) < 1e-12
            assert [[list(a), list(b)] for a, b in layouts] == d["layouts"]
            assert len(switches) == len(d["switches"])
            for got, want in zip(switches, d["switches"]):
                for key in ("from", "to", "runs", "messages", "bytes_remote", "bytes_resident"):
                    assert got[key] == want[key], key


def test_bundled_and_multilevel_match_reference(golden):
    docs, states = golden.json("bundled"), golden.npz("bundled")
    for name, doc in docs.items():
        c = parse_qasm(doc["qasm"])
        ref = states[name]
        assert np.max(np.abs(orc.simulate_flat(c) - ref)) < 1e-12
        for parts in doc["partitions"].values():
            assert np.max(np.abs(orc.execute_hierarchical(c, parts_of(parts)) - ref)) < 1e-12
        if "multilevel" in doc:
            ml = doc["multilevel"]
            got = orc.execute_multilevel(c, parts_of(ml["level1"]), [parts_of(s) for s in ml["sublevels"]],
                                         ml["padded"])
            assert np.max(np.abs(got - ref)) < 1e-12


def _sample_check(golden, name, psi):
    doc = golden.json("configs")[name + ":sample"]
    arr = golden.npz("configs")
    key = name.replace("@", "_")
    idx, amp = arr[key + "_idx"], arr[key + "_amp"]
    assert np.max(np.abs(psi[idx] - amp)) < 1e-12
    assert abs(np.linalg.norm(psi) - doc["norm"]) < 1e-12


def test_c1_numpy_oracle_and_closed_form(golden):
    doc = golden.json("configs")["c1:sample"]
    c = configs.build("c1")
    psi = orc.execute_hierarchical(c, parts_of(doc["partition"]))
    _sample_check(golden, "c1", psi)
    x = configs.qft_prefix_index(20, 0)
    idx = golden.npz("configs")["c1_idx"]
    closed = orc.qft_basis_amplitudes(20, x, idx)
    assert np.max(np.abs(closed - psi[idx])) < 1e-12


@pytest.mark.parametrize("name", ["c2@20", "c3@20", "c4@small18"])
def test_c_oracle_matches_reference_samples(golden, name):
    doc = golden.json("configs")[name + ":sample"]
    c = configs.ising_config(18, 4) if name == "c4@small18" else configs.build(name)
    psi = c_oracle.execute_parts(c, parts_of(doc["partition"]))
    _sample_check(golden, name, psi)


@pytest.mark.parametrize("name,fixture", [("c2@24", "configs_large"), ("c3@24", "configs_large"),
                                          ("c4@22", "configs_large_c4")])
def test_c_oracle_matches_reference_samples_at_24_qubits(golden, name, fixture):
    """The C oracle against the unmodified reference at 24 qubits
    (tests/golden/make_golden_large.py): sampled amplitudes, norm, and the
    weighted checksum over every |amp|^2."""
    doc = golden.json(fixture)[name + ":sample"]
    arr = golden.npz(fixture)
    key = name.replace("@", "_")
    c = configs.build(name)
    psi = c_oracle.execute_parts(c, parts_of(doc["partition"]))
    assert np.max(np.abs(psi[arr[key + "_idx"]] - arr[key + "_amp"])) < 1e-12
    p2 = psi.real ** 2 + psi.imag ** 2
    assert abs(np.sqrt(p2.sum()) - doc["norm"]) < 1e-12
    assert abs(float(np.sum(p2 * (np.arange(p2.size) % 7))) - doc["checksum_abs2_weighted"]) < 1e-10


def test_c_oracle_matches_corpus_and_flat(golden):
    docs, states = golden.json("corpus"), golden.npz("corpus")
    for i, doc in enumerate(docs[:30]):
        c = parse_qasm(doc["qasm"])
        assert np.max(np.abs(c_oracle.simulate_flat(c) - states[f"c{i}"])) < 1e-12
        for parts in list(doc["partitions"].values())[:3]:
            got = c_oracle.execute_parts(c, parts_of(parts))
            assert np.max(np.abs(got - states[f"c{i}"])) < 1e-12


def test_c_oracle_sampled_fixings_compose():
    """Running a part over fixing ranges in pieces equals one full pass."""
    c = configs.build("c2@14")
    from paper_2205_06973_b200 import build_dag, partition_dfs

    part = partition_dfs(build_dag(c), 8).parts[0]
    pos, ops, slots = c_oracle.part_slots(c, part.gate_indices, part.qubits)
    rng = np.random.default_rng(1)
    psi = rng.normal(size=1 << 14) + 1j * rng.normal(size=1 << 14)
    a, b = psi.copy(), psi.copy()
    c_oracle.run_part(a, pos, ops, slots)
    total = 1 << (14 - len(pos))
    c_oracle.run_part(b, pos, ops, slots, 0, total // 3)
    c_oracle.run_part(b, pos, ops, slots, total // 3, total - total // 3)
    np.testing.assert_array_equal(a, b)


def test_memory_formula():
    from paper_2205_06973_b200.statevec import state_bytes

    assert all(state_bytes(n) == 1 << (n + 4) for n in range(0, 51))
    assert state_bytes(30) == 17_179_869_184
    assert math.isclose(state_bytes(20, "complex64"), 8 << 20)
