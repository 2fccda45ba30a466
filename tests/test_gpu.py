"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle
and the reference's golden vectors. Tolerances are the north star's:
max-abs 1e-10 for complex128, 1e-4 for complex64."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import parts_of, partition_of  # noqa: E402
from oracle import c_oracle  # noqa: E402
from oracle import hisim_oracle as orc  # noqa: E402
from paper_2205_06973_b200 import (  # noqa: E402
    _native,
    build_dag,
    configs,
    execute_hierarchical,
    execute_multilevel,
    partition_dagp,
    partition_dfs,
    partition_multilevel,
    partition_nat,
    simulate_distributed,
)
from paper_2205_06973_b200.errors import PartTooWideForLayoutError  # noqa: E402
from paper_2205_06973_b200.hier import HierarchicalRun, max_abs_diff, remap_part, run_part  # noqa: E402
from paper_2205_06973_b200.qasm import GateKind, GateOp, parse_qasm  # noqa: E402
from paper_2205_06973_b200.statevec import apply_gate, from_numpy, simulate_flat  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"complex128": 1e-10, "complex64": 1e-4}


def _dev_err(state, ref):
    return float(np.max(np.abs(state.to_numpy() - ref)))


@pytest.mark.parametrize("dtype,merge", [("complex128", True), ("complex64", True), ("complex128", False)])
def test_corpus_every_partition_matches_reference(golden, dtype, merge, monkeypatch):
    """Every corpus circuit under every reference partition; with the
    default HS_PLAN_MERGE (consecutive parts that fit one tile share a pass)
    and without it (one pass per part)."""
    if not merge:
        monkeypatch.setattr(_native, "_default_options", _native.default_options() & ~_native.HS_PLAN_MERGE)
    docs, states = golden.json("corpus"), golden.npz("corpus")
    worst = 0.0
    for i, doc in enumerate(docs):
        c = parse_qasm(doc["qasm"])
        for key, parts in doc["partitions"].items():
            st = execute_hierarchical(c, partition_of(parts), dtype=dtype)
            worst = max(worst, _dev_err(st, states[f"c{i}"]))
    assert worst < TOL[dtype], worst


def test_bundled_multilevel_and_traces(golden):
    docs, states = golden.json("bundled"), golden.npz("bundled")
    for name, doc in docs.items():
        c = parse_qasm(doc["qasm"])
        d = build_dag(c)
        for strategy, parts in doc["partitions"].items():
            st = execute_hierarchical(c, partition_of(parts))
            assert _dev_err(st, states[name]) < 1e-10, (name, strategy)
        _, tr = execute_hierarchical(c, partition_nat(d, doc["limit"]), with_trace=True)
        assert tr.part_rows() == doc["nat_trace"]
        if "multilevel" in doc:
            ml = doc["multilevel"]
            part = partition_multilevel(d, ml["limit1"], ml["limit2"])
            st, tr = execute_multilevel(c, part, with_trace=True)
            assert _dev_err(st, states[name]) < 1e-10
            assert tr.part_rows() == ml["trace"]


def test_flat_and_single_gates(golden):
    docs, states = golden.json("corpus"), golden.npz("corpus")
    for i, doc in enumerate(docs[:20]):
        c = parse_qasm(doc["qasm"])
        assert _dev_err(simulate_flat(c, max_qubits=c.num_qubits), states[f"c{i}"]) < 1e-10
    # apply_gate on a random state, every gate kind, vs the oracle
    rng = np.random.default_rng(3)
    n = 7
    raw = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    for kind in GateKind:
        qubits = tuple(int(x) for x in rng.choice(n, kind.arity, replace=False))
        op = GateOp(kind, qubits, tuple(float(x) for x in rng.uniform(-3, 3, kind.num_params)))
        sv = from_numpy(raw)
        apply_gate(sv, op)
        want = raw.copy()
        orc.apply_op(want, n, op)
        assert _dev_err(sv, want) < 1e-12, kind


def test_run_part_api_numpy_torch_and_batches():
    c = configs.build("c2@12")
    part = partition_dfs(build_dag(c), 9).parts[1]
    exe = remap_part(c, part)
    rng = np.random.default_rng(0)
    data = rng.normal(size=(4, 1 << 12)) + 1j * rng.normal(size=(4, 1 << 12))
    want = data.copy()
    orc.run_part(want, exe.slot_map.qubits, exe.ops, exe.op_slots)
    host = data.copy()
    run_part(host, exe)  # numpy in, numpy out (copied through the device)
    assert np.max(np.abs(host - want)) < 1e-12
    dev = torch.from_numpy(data.copy()).cuda()
    run_part(dev, exe)
    assert np.max(np.abs(dev.cpu().numpy() - want)) < 1e-12
    with pytest.raises(ValueError):
        run_part(torch.zeros(3, dtype=torch.complex128, device="cuda"), exe)


def _sample(golden, name, st):
    arr = golden.npz("configs")
    key = name.replace("@", "_")
    idx, amp = arr[key + "_idx"], arr[key + "_amp"]
    got = st.data[torch.as_tensor(idx, device=st.data.device)].cpu().numpy()
    return float(np.max(np.abs(got - amp)))


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_config1_qft_full_state_closed_form(golden, dtype):
    """c1 at full size: sampled reference amplitudes, and every one of the
    2^20 amplitudes against the closed-form QFT of the prepared basis state."""
    c = configs.build("c1")
    for strategy in ("nat", "dfs", "dagp"):
        part = {"nat": partition_nat, "dfs": partition_dfs, "dagp": partition_dagp}[strategy](build_dag(c), 10)
        st = execute_hierarchical(c, part, dtype=dtype)
        assert _sample(golden, "c1", st) < TOL[dtype]
        x = configs.qft_prefix_index(20, 0)
        ks = np.arange(1 << 20)
        rev = np.zeros_like(ks)
        for b in range(20):
            rev |= ((ks >> b) & 1) << (19 - b)
        rx = int(sum(((x >> b) & 1) << (19 - b) for b in range(20)))
        closed = np.exp(2j * np.pi * ((rx * rev) % (1 << 20)) / (1 << 20)) / 1024.0
        assert max_abs_diff(st, closed) < TOL[dtype]


@pytest.mark.parametrize("name", ["c2@20", "c3@20", "c4@small18"])
def test_scaled_configs_match_reference_samples(golden, name):
    doc = golden.json("configs")[name + ":sample"]
    c = configs.ising_config(18, 4) if name == "c4@small18" else configs.build(name)
    st = execute_hierarchical(c, partition_of(doc["partition"]))
    assert _sample(golden, name, st) < 1e-10
    assert abs(st.norm() - doc["norm"]) < 1e-10


@pytest.mark.parametrize("name,fixture", [("c2@24", "configs_large"), ("c3@24", "configs_large"),
                                          ("c4@22", "configs_large_c4")])
def test_24_qubit_programs_match_the_reference_itself(golden, name, fixture):
    """The compiled paths against the UNMODIFIED reference's own amplitudes
    (no oracle in between) at the largest size the reference runs in minutes:
    24-qubit c2 / c3 and 22-qubit c4 (tests/golden/make_golden_large.py ran hier.py:342-368
    there; 4096 sampled amplitudes, the norm and a weighted checksum of every
    |amp|^2). Checked: execute_hierarchical, the program bench.py times
    (|0..0> in its own initial layout, ping-pong passes, one CUDA graph), the
    one-pass-per-part program and simulate_distributed over 2 and 8 ranks."""
    from paper_2205_06973_b200.statevec import StateVector, allocate

    doc = golden.json(fixture)[name + ":sample"]
    arr = golden.npz(fixture)
    key = name.replace("@", "_")
    c = configs.build(name)
    n = c.num_qubits
    assert (n, c.num_ops) == (doc["num_qubits"], doc["num_ops"])
    part = partition_of(doc["partition"], "dfs", doc["limit"])
    idx = torch.as_tensor(arr[key + "_idx"], device="cuda")
    weights = (torch.arange(1 << n, device="cuda") % 7).to(torch.float64)

    def check(data, tol=1e-10):
        got = data[idx].cpu().numpy()
        assert float(np.max(np.abs(got - arr[key + "_amp"]))) < tol
        p2 = data.real.double() ** 2 + data.imag.double() ** 2
        assert abs(float(p2.sum().sqrt()) - doc["norm"]) < tol
        assert abs(float((p2 * weights).sum()) - doc["checksum_abs2_weighted"]) < 10 * tol

    check(execute_hierarchical(c, part).data)
    # any valid partition ends in the same state: this repo's dagP parts, and complex64 at the north star's 1e-4
    check(execute_hierarchical(c, partition_dagp(build_dag(c), doc["limit"])).data)
    check(execute_hierarchical(c, part, dtype="complex64").data, TOL["complex64"])
    # parts wider than one 12-qubit tile (k = 14, the c5 path) and the two-level run (hier.py:371-419)
    check(execute_hierarchical(c, partition_dfs(build_dag(c), 14)).data)
    check(execute_multilevel(c, partition_multilevel(build_dag(c), doc["limit"], 8)).data)
    buf = allocate(n)
    timed = HierarchicalRun(c, part, basis_start=True)
    assert all(timed.program.info(j)["compiled"] for j in range(timed.program.num_launches))
    for _ in range(2):  # graph capture, then replay
        timed.program.init_basis(buf, 0)
        timed.program.run_graph(buf)
        check(StateVector(n, buf).data)
    literal = HierarchicalRun(c, part, basis_start=True, options=(timed.program.options & ~_native.HS_PLAN_MERGE)
                              | _native.HS_PLAN_PART_LOCAL)
    literal.program.init_basis(buf, 0)
    literal.program.run_graph(buf)
    check(StateVector(n, buf).data)
    del buf, timed, literal
    # the sharded path (emulated ranks on this GPU, dist.py:485-529) ends in the same state
    for p_bits in (1, 3):
        check(simulate_distributed(c, part, p_bits).state.data)


@pytest.mark.parametrize("name,strategy", [("c2", "dfs"), ("c2", "dagp"), ("c3@26", "dfs")])
def test_full_size_configs_match_c_oracle(golden, name, strategy):
    """26-qubit runs against the multi-threaded C oracle (same partition)."""
    c = configs.build(name)
    d = build_dag(c)
    part = (partition_dfs if strategy == "dfs" else partition_dagp)(d, 12)
    st = execute_hierarchical(c, part)
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    assert max_abs_diff(st, ref) < 1e-10


@pytest.mark.parametrize("name,strategy,force", [("c2@24", "dfs", True), ("c2@24", "dagp", True),
                                                 ("c4@26", "dfs", False), ("c3@26", "dagp", False),
                                                 ("c1", "dfs", False)])
def test_global_diagonal_programs_match_c_oracle(name, strategy, force, monkeypatch):
    """Compiled passes with global (unstaged) diagonal qubits: CZs with a
    global control or target (random circuits, forced with
    HISVSIM_GLOBAL_DIAG=1), parity diagonals of CX.RZ.CX (c3 / c4) and
    CRZ / U1 (c1) whose values come from the tile's free index bits; the
    programs must carry global passes and equal the C oracle."""
    import ctypes

    from paper_2205_06973_b200.hier import PartProgram, _pack

    if force:
        monkeypatch.setenv("HISVSIM_GLOBAL_DIAG", "1")
    c = configs.build(name)
    part = (partition_dfs if strategy == "dfs" else partition_dagp)(build_dag(c), 12)
    exes = [remap_part(c, p) for p in part.parts]
    prog = PartProgram(c.num_qubits, exes)
    lib = _native.load()
    parts, gates, total = _pack(exes)
    size, nl = ctypes.c_size_t(), ctypes.c_int()
    _native.check(lib.hs_plan_program(c.num_qubits, 0, 12, prog.options, parts, len(exes), gates, total, None, 0,
                                      ctypes.byref(size), ctypes.byref(nl)))
    buf = ctypes.create_string_buffer(size.value)
    _native.check(lib.hs_plan_program(c.num_qubits, 0, 12, prog.options, parts, len(exes), gates, total, buf,
                                      size.value, ctypes.byref(size), ctypes.byref(nl)))
    raw, off, globals_ = buf.raw, 0, 0
    for _ in range(nl.value):
        nprog = int.from_bytes(raw[off + 8:off + 12], "little", signed=True)
        first_op = int.from_bytes(raw[off + 144:off + 146], "little") if nprog else 0
        globals_ += first_op == 5
        off += 144 + 96 * nprog
    assert globals_ > 0
    st = execute_hierarchical(c, part)
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    assert max_abs_diff(st, ref) < 1e-10


def test_global_diagonal_edge_circuits_on_gpu(monkeypatch):
    """Compiled passes on 22 qubits for the emulated edge cases: a graph
    state (CZs with both qubits unstaged) and a circuit of diagonal gates
    only (passes that stage nothing), against the C oracle."""
    import random

    from paper_2205_06973_b200.qasm import Circuit

    monkeypatch.setenv("HISVSIM_GLOBAL_DIAG", "1")
    rng = random.Random(3)
    n = 22
    graph = [GateOp(GateKind.H, (q,), ()) for q in range(n)]
    graph += [GateOp(GateKind.CZ, (a, b), ()) for a in range(n) for b in range(a + 1, n) if (a * 5 + b) % 4 == 0]
    graph += [GateOp(GateKind.RX, (q,), (0.2 + 0.1 * q,)) for q in range(n)]
    diag = [GateOp(GateKind.H, (q,), ()) for q in range(0, n, 3)]
    for _ in range(200):
        a, b = rng.sample(range(n), 2)
        k = rng.choice([GateKind.T, GateKind.RZ, GateKind.CZ, GateKind.CRZ])
        diag.append(GateOp(k, (a, b) if k in (GateKind.CZ, GateKind.CRZ) else (a,),
                           (rng.uniform(0, 3),) if k in (GateKind.RZ, GateKind.CRZ) else ()))
    for ops in (graph, diag):
        c = Circuit(n, tuple(ops))
        part = partition_dfs(build_dag(c), 10)
        st = execute_hierarchical(c, part)
        ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
        assert max_abs_diff(st, ref) < 1e-10


@pytest.mark.parametrize("name", ["c4@24", "c3@24"])
def test_global_diagonal_programs_complex64(name):
    """complex64 compiled passes with global diagonals (the gw word and the
    gq / gc masks in the float kernels) against the C oracle at 1e-4."""
    c = configs.build(name)
    part = partition_dfs(build_dag(c), 12)
    st = execute_hierarchical(c, part, dtype="complex64")
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    assert max_abs_diff(st, ref) < 1e-4


def test_distributed_emulated_ranks_match_reference(golden):
    docs, states = golden.json("corpus"), golden.npz("corpus")
    for i, doc in enumerate(docs):
        c = parse_qasm(doc["qasm"])
        for d in doc["dist"]:
            run = simulate_distributed(c, partition_of(d["parts"]), d["p"])
            assert _dev_err(run.state, states[f"c{i}"]) < 1e-10
            assert [[list(l.local), list(l.process)] for l in run.layouts] == d["layouts"]
            assert [s.bytes_remote for s in run.stats.switches] == [s["bytes_remote"] for s in d["switches"]]


def test_distributed_c1_at_three_rank_bits(golden):
    c = configs.build("c1")
    part = partition_dagp(build_dag(c), 10)
    run = simulate_distributed(c, part, 3)
    assert _sample(golden, "c1", run.state) < 1e-10


def test_program_reuse_graph_and_initial_state():
    c = configs.build("c2@16")
    part = partition_dfs(build_dag(c), 10)
    run = HierarchicalRun(c, part)
    rng = np.random.default_rng(9)
    raw = rng.normal(size=1 << 16) + 1j * rng.normal(size=1 << 16)
    raw /= np.linalg.norm(raw)
    want = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in part.parts], initial=raw)
    a = from_numpy(raw)
    run.program.run(a.data)
    b = from_numpy(raw)
    run.program.run_graph(b.data)
    run.program.run_graph(b.data)  # replay: applies the circuit twice
    twice = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in part.parts], initial=want)
    assert _dev_err(a, want) < 1e-10
    assert _dev_err(b, twice) < 1e-10


def test_layout_kernels_round_trip():
    import ctypes

    lib = _native.load()
    n = 14
    x = torch.randn(1 << n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    perm = list(range(n))
    np.random.default_rng(2).shuffle(perm)
    inv = [perm.index(b) for b in range(n)]
    s = torch.cuda.current_stream().cuda_stream
    _native.check(lib.hs_bit_permute(x.data_ptr(), y.data_ptr(), n, 0, (ctypes.c_int32 * n)(*perm), s))
    _native.check(lib.hs_bit_permute(y.data_ptr(), z.data_ptr(), n, 0, (ctypes.c_int32 * n)(*inv), s))
    assert torch.equal(x, z)
    idx = torch.arange(1 << n, device="cuda")
    moved = torch.zeros(1 << n, dtype=torch.long, device="cuda")
    dst = torch.zeros_like(idx)
    for b in range(n):
        dst |= ((idx >> b) & 1) << perm[b]
    assert torch.equal(y[dst], x)
    seg = (ctypes.c_int32 * 3)(2, 5, 11)
    _native.check(lib.hs_pack_segments(x.data_ptr(), y.data_ptr(), n, 0, seg, 3, s))
    _native.check(lib.hs_unpack_segments(y.data_ptr(), z.data_ptr(), n, 0, seg, 3, s))
    assert torch.equal(x, z)
    del moved


def test_errors_surface_as_reference_exceptions():
    from paper_2205_06973_b200.qasm import Circuit

    c = Circuit(16, tuple(GateOp(GateKind.H, (q,)) for q in range(16)))
    part = partition_of([(list(range(16)), list(range(16)))], limit=16)
    # wider than any tile: runs as sub-passes (no error), H^16 |0> is uniform
    st = execute_hierarchical(c, part)
    assert float(np.max(np.abs(st.to_numpy() - 2.0 ** -8))) < 1e-12
    # wider than the ranks' local qubits: the reference's layout error (dist.py:136-141)
    with pytest.raises(PartTooWideForLayoutError):
        simulate_distributed(c, part, 1)


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_compiled_parts_match_reference(golden, dtype):
    """HS_PLAN_JIT (NVRTC straight-line kernels) on corpus circuits, the full
    c1 QFT and scaled c2/c3 against the reference's results."""
    from paper_2205_06973_b200.hier import PartProgram

    opts = _native.default_options() | _native.HS_PLAN_JIT
    docs, states = golden.json("corpus"), golden.npz("corpus")
    for i, doc in enumerate(docs[:12]):
        c = parse_qasm(doc["qasm"])
        key = sorted(doc["partitions"])[0]
        part = partition_of(doc["partitions"][key])
        exes = [remap_part(c, p) for p in part.parts]
        prog = PartProgram(c.num_qubits, exes, dtype=dtype, options=opts)
        assert prog.jit_error == "" and all(prog.info(j)["compiled"] for j in range(prog.num_launches))
        st = from_numpy(np.eye(1, 1 << c.num_qubits, 0).ravel().astype(np.complex128), dtype=dtype)
        prog.run(st.data)
        assert _dev_err(st, states[f"c{i}"]) < TOL[dtype]
    for name in ("c2@20", "c3@20"):
        doc = golden.json("configs")[name + ":sample"]
        c = configs.build(name)
        st = execute_hierarchical(c, partition_of(doc["partition"]), dtype=dtype)  # n >= 20: compiled
        assert _sample(golden, name, st) < TOL[dtype]


def test_compiled_full_size_c2_matches_c_oracle():
    c = configs.build("c2")
    part = partition_dfs(build_dag(c), 12)
    run = HierarchicalRun(c, part)
    assert all(run.program.info(j)["compiled"] for j in range(run.program.num_launches))
    from paper_2205_06973_b200.statevec import zero_state

    st = zero_state(26)
    run.program.run(st.data)
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    assert max_abs_diff(st, ref) < 1e-10


@pytest.mark.parametrize("name", ["c3@24", "c2@24"])
def test_initial_layout_for_basis_starts(name):
    """HS_PLAN_INIT_LAYOUT: a program that only ever starts from basis states
    picks its own initial layout (part 0's qubits lowest); |x> prepared with
    init_basis in that layout gives the natural-order result of |x>."""
    from paper_2205_06973_b200.statevec import allocate

    c = configs.build(name)
    part = partition_dfs(build_dag(c), 12)
    run = HierarchicalRun(c, part, basis_start=True)
    n = c.num_qubits
    assert run.program.initial_layout != tuple(range(n))
    assert sorted(run.program.initial_layout) == list(range(n))
    x = 0b1011001110001011010110 & ((1 << n) - 1)
    st = allocate(n)
    run.program.init_basis(st, x)
    run.program.run(st)
    init = np.zeros(1 << n, dtype=np.complex128)
    init[x] = 1.0
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts], initial=init)
    assert float(np.max(np.abs(st.cpu().numpy() - ref))) < 1e-10
    # a caller's natural-order state goes through a program without one
    plain = HierarchicalRun(c, part, basis_start=False)
    assert plain.program.initial_layout == tuple(range(n))


@pytest.mark.parametrize("name,limit,dtype", [("c2@22", 14, "complex128"), ("c2@24", 13, "complex128"),
                                              ("c2@17", 14, "complex128"), ("c2@22", 14, "complex64")])
def test_wide_parts_match_c_oracle(name, limit, dtype):
    """c5's k = 14 parts (256 KB of complex128 per tile, more than one SM
    holds): by default sub-passes that fit the tile; with HS_PLAN_CLUSTER
    one pass over a 2-4 CTA cluster sharing the tile through distributed
    shared memory. Sub-passes regroup the whole gate stream by default,
    per part with HS_PLAN_PART_LOCAL."""
    c = configs.build(name)
    part = partition_dfs(build_dag(c), limit)
    assert max(len(p.qubits) for p in part.parts) == limit
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    base = _native.default_options() | _native.HS_PLAN_JIT | _native.HS_PLAN_LAYOUT
    for opts in (None, base | _native.HS_PLAN_PART_LOCAL, base | _native.HS_PLAN_CLUSTER,
                 base | _native.HS_PLAN_CLUSTER | _native.HS_PLAN_PINGPONG):
        run = HierarchicalRun(c, part, dtype=dtype, options=opts)
        assert run.program.jit_error == ""
        owners = [run.program.info(j)["user_part"] for j in range(run.program.num_launches)]
        if opts is None:  # regrouped passes: a pass may carry two parts' gates
            assert set(u for u in owners if u >= 0) <= set(range(part.num_parts))
        else:
            assert sorted(set(u for u in owners if u >= 0)) == list(range(part.num_parts))
        st = from_numpy(np.eye(1, 1 << c.num_qubits, 0).ravel().astype(np.complex128), dtype=dtype)
        run.program.run(st.data)
        assert float(np.max(np.abs(st.to_numpy() - ref))) < TOL[dtype], opts


def test_segment_range_pack_unpack_kernels():
    """hs_pack/unpack_segments_range (the in-place switch's chunk moves)
    against numpy index arithmetic, complex128 and complex64."""
    from paper_2205_06973_b200.multi import DeviceOps

    ops = DeviceOps()
    rng = np.random.default_rng(3)
    for dt in (torch.complex128, torch.complex64):
        n, seg_pos = 14, [2, 7, 11]
        src = torch.tensor(rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n), dtype=dt, device="cuda")
        inner = 1 << (n - len(seg_pos))
        begin, cnt = 37, 300
        st = torch.empty(cnt << len(seg_pos), dtype=dt, device="cuda")
        ops.pack_range(src, st, n, seg_pos, begin, cnt)
        host = src.cpu().numpy()
        for k in range(1 << len(seg_pos)):
            m = np.arange(begin, begin + cnt)
            idx = m.copy()
            for b, q in enumerate(seg_pos):
                lo = idx & ((1 << q) - 1)
                idx = ((idx ^ lo) << 1) | lo | (((k >> b) & 1) << q)
            assert np.array_equal(st[k * cnt:(k + 1) * cnt].cpu().numpy(), host[idx])
        dst = torch.zeros_like(src)
        ops.unpack_range(st, dst, n, seg_pos, begin, cnt)
        back = torch.zeros_like(st)
        ops.pack_range(dst, back, n, seg_pos, begin, cnt)
        assert torch.equal(back, st)
        assert inner > begin + cnt


def test_program_from_a_given_layout():
    """A program fed a buffer in an arbitrary physical layout (what an
    in-place switch leaves) ends in natural order with the right amplitudes."""
    from paper_2205_06973_b200.hier import PartProgram
    from paper_2205_06973_b200.statevec import allocate

    c = configs.build("c3@24")
    part = partition_dfs(build_dag(c), 12)
    exes = [remap_part(c, p) for p in part.parts]
    n = c.num_qubits
    rng = np.random.default_rng(11)
    phys = [int(x) for x in rng.permutation(n)]
    init = np.zeros(1 << n, dtype=np.complex128)
    init[rng.integers(0, 1 << n, 64)] = rng.standard_normal(64)
    init /= np.linalg.norm(init)
    # natural -> physical: logical index i sits at sum_q bit_q(i) << phys[q]
    i = np.arange(1 << n, dtype=np.int64)
    dst = np.zeros_like(i)
    for q, b in enumerate(phys):
        dst |= ((i >> q) & 1) << b
    buf = np.zeros_like(init)
    buf[dst] = init
    prog = PartProgram(n, exes, init_layout=phys)
    st = torch.from_numpy(buf).cuda()
    prog.run(st)
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts], initial=init)
    assert float(np.max(np.abs(st.cpu().numpy() - ref))) < 1e-10


@pytest.mark.parametrize("policy", ["reference", "lookahead"])
def test_sharded_run_loopback_on_one_gpu(golden, policy):
    """The distributed path's device pieces - in-place chunked switches
    (pack/unpack kernels) and segment programs starting from the arrival
    layout - for all ranks on one GPU (transfers as copies), against the
    reference's distributed results on the corpus."""
    from paper_2205_06973_b200.multi import ShardedRun, run_loopback, shard_positions

    docs, states = golden.json("corpus"), golden.npz("corpus")
    checked = handed = 0
    for i, doc in enumerate(docs):
        c = parse_qasm(doc["qasm"])
        for d in doc["dist"]:
            if not d["switches"] or c.num_qubits < 8:
                continue
            run = ShardedRun(c, partition_of(d["parts"]), d["p"], loopback=True, chunk_bytes=256, policy=policy)
            if policy == "reference":
                assert [[list(x.local), list(x.process)] for x in run.layouts] == d["layouts"]
            R = 1 << d["p"]
            shards = [torch.zeros(1 << run.n_local, dtype=torch.complex128, device="cuda") for _ in range(R)]
            shards[0][0] = 1.0
            shards = run_loopback(run, shards)
            full = np.zeros(1 << c.num_qubits, dtype=np.complex128)
            for r in range(R):
                full[shard_positions(run.layouts[-1], r)] = shards[r].cpu().numpy()
            assert np.max(np.abs(full - states[f"c{i}"])) < 1e-10, (i, d["p"])
            checked += 1
            handed += sum(1 for ph in run.seg_phys_out[:-1] if ph is not None)
    assert checked >= 5
    assert handed >= 1  # some switch packed straight from a segment's final (non-natural) layout


def test_run_stream_many_initial_states():
    """HierarchicalRun.run_stream: several host initial states through the
    overlapped upload / parts / download pipeline, each against the oracle."""
    c = configs.build("c2@20")
    part = partition_dfs(build_dag(c), 12)
    run = HierarchicalRun(c, part, basis_start=False)
    n = c.num_qubits
    rng = np.random.default_rng(5)
    ins, outs, refs = [], [], []
    parts = [(p.gate_indices, p.qubits) for p in part.parts]
    for k in range(5):
        x = np.zeros(1 << n, dtype=np.complex128)
        x[rng.integers(0, 1 << n, 3)] = rng.standard_normal(3)
        x /= np.linalg.norm(x)
        ins.append(torch.from_numpy(x).pin_memory())
        outs.append(torch.empty(1 << n, dtype=torch.complex128).pin_memory())
        refs.append(c_oracle.execute_parts(c, parts, initial=x))
    run.run_stream(ins, outs)
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert float(np.max(np.abs(o.numpy() - r))) < 1e-10


@pytest.mark.parametrize("extra,dtype", [("layout", "complex128"), ("pingpong", "complex128"),
                                         ("pingpong_init", "complex128"), ("cluster", "complex128"),
                                         ("pingpong_init", "complex64"), ("merged", "complex128")])
def test_corpus_through_every_compiled_path(golden, extra, dtype):
    """Every corpus circuit and partition (all gate kinds, controls on thread
    and register bits, SWAPs, tiny states where a team is a few threads)
    through the compiled kernels with the layout machinery switched on."""
    from paper_2205_06973_b200.hier import PartProgram

    base = (_native.default_options() & ~_native.HS_PLAN_MERGE) | _native.HS_PLAN_JIT  # one pass per part
    opts = {"merged": base | _native.HS_PLAN_MERGE | _native.HS_PLAN_LAYOUT | _native.HS_PLAN_PINGPONG,
            "layout": base | _native.HS_PLAN_LAYOUT,
            "pingpong": base | _native.HS_PLAN_LAYOUT | _native.HS_PLAN_PINGPONG,
            "pingpong_init": base | _native.HS_PLAN_LAYOUT | _native.HS_PLAN_PINGPONG | _native.HS_PLAN_INIT_LAYOUT,
            "cluster": base | _native.HS_PLAN_CLUSTER}[extra]
    docs, states = golden.json("corpus"), golden.npz("corpus")
    checked = 0
    for i, doc in enumerate(docs):
        if i % 4:  # every fourth circuit, all its partitions (NVRTC compiles every part)
            continue
        c = parse_qasm(doc["qasm"])
        for key, parts in doc["partitions"].items():
            part = partition_of(parts)
            exes = [remap_part(c, p) for p in part.parts]
            prog = PartProgram(c.num_qubits, exes, options=opts, dtype=dtype)
            assert prog.jit_error == ""
            st = torch.zeros(1 << c.num_qubits, dtype=prog.dtype, device="cuda")
            prog.init_basis(st, 0)
            prog.run(st)
            err = float(np.max(np.abs(st.cpu().numpy().astype(np.complex128) - states[f"c{i}"])))
            assert err < TOL[dtype], (i, key, extra)
            checked += 1
    assert checked >= 15


def test_emulated_ranks_lookahead_policy(golden):
    """simulate_distributed(policy="lookahead"): the same amplitudes as the
    reference with no more remote bytes than its schedule."""
    docs, states = golden.json("corpus"), golden.npz("corpus")
    for i, doc in enumerate(docs[:20]):
        c = parse_qasm(doc["qasm"])
        for d in doc["dist"]:
            run = simulate_distributed(c, partition_of(d["parts"]), d["p"], policy="lookahead")
            assert _dev_err(run.state, states[f"c{i}"]) < 1e-10
            assert run.stats.total_bytes <= sum(s["bytes_remote"] for s in d["switches"])


@pytest.mark.parametrize("policy", ["reference", "lookahead"])
def test_sharded_run_loopback_large_shards(policy):
    """24 qubits over 2 ranks (23 local: compiled, layout-planned segments):
    segments before a switch end in their own layout and the switch packs
    from it; the assembled state equals the C oracle's."""
    from paper_2205_06973_b200.multi import ShardedRun, run_loopback, shard_positions

    c = configs.build("c3@24")
    part = partition_dfs(build_dag(c), 12)
    run = ShardedRun(c, part, 1, loopback=True, policy=policy)
    assert run.switch_at
    shards = [torch.zeros(1 << run.n_local, dtype=torch.complex128, device="cuda") for _ in range(2)]
    shards[0][0] = 1.0
    shards = run_loopback(run, shards)
    full = np.zeros(1 << c.num_qubits, dtype=np.complex128)
    for r in range(2):
        full[shard_positions(run.layouts[-1], r)] = shards[r].cpu().numpy()
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    assert float(np.max(np.abs(full - ref))) < 1e-10
    assert any(ph is not None for ph in run.seg_phys_out[:-1])
    # the segment programs share one ping-pong scratch buffer
    scratch = {id(pr._scratch) for pr in run.programs if pr is not None and pr.needs_scratch}
    assert len(scratch) <= 1


def test_edge_case_circuits():
    """Empty circuits, one qubit, SWAP-only circuits (no arithmetic: pure
    relabels) and a single wide CCX, through the compiled path (n >= 20) and
    the interpreter, against the oracle."""
    from paper_2205_06973_b200.qasm import Circuit

    def check(c, limit):
        part = partition_dfs(build_dag(c), limit)
        st = execute_hierarchical(c, part)
        ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
        assert float(np.max(np.abs(st.to_numpy() - ref))) < 1e-12
        return part.num_parts

    assert check(Circuit(21, ()), 12) == 0
    check(Circuit(1, (GateOp(GateKind.H, (0,)),)), 1)
    swaps = tuple(GateOp(GateKind.SWAP, (a, b)) for a, b in [(0, 20), (3, 17), (20, 5), (1, 2), (19, 0)])
    check(Circuit(21, (GateOp(GateKind.X, (0,)), GateOp(GateKind.H, (3,))) + swaps), 12)
    check(Circuit(22, (GateOp(GateKind.X, (0,)), GateOp(GateKind.X, (21,)),
                       GateOp(GateKind.CCX, (0, 21, 11)), GateOp(GateKind.SWAP, (11, 1)))), 3)


def _inverse_appended(c):
    """The circuit followed by its inverse (reversed ops, each inverted within
    the reference gate set): the product is the identity, so a basis start
    must come back exactly - a size-independent check at full config sizes."""
    from paper_2205_06973_b200.qasm import Circuit

    swap = {GateKind.S: GateKind.SDG, GateKind.SDG: GateKind.S, GateKind.T: GateKind.TDG, GateKind.TDG: GateKind.T}
    angle = {GateKind.RX, GateKind.RY, GateKind.RZ, GateKind.U1, GateKind.CRZ, GateKind.CRY}
    inv = []
    for op in reversed(c.ops):
        if op.kind in swap:
            inv.append(GateOp(swap[op.kind], op.qubits, ()))
        elif op.kind in angle:
            inv.append(GateOp(op.kind, op.qubits, (-op.params[0],)))
        elif op.kind == GateKind.U3:  # U3(t, p, l)^-1 = U3(-t, -l, -p)
            t, p, l = op.params
            inv.append(GateOp(op.kind, op.qubits, (-t, -l, -p)))
        else:  # H, X, Y, Z, CX, CZ, SWAP, CCX are their own inverses
            inv.append(op)
    return Circuit(c.num_qubits, tuple(c.ops) + tuple(inv))


def _basis_error(state, index):
    """max |psi - e_index| over the device state, in chunks (33-qubit states
    leave no room for a full-size temporary)."""
    d = state.data
    worst = abs(complex(d[index].item()) - 1.0)
    step = 1 << 26
    for s in range(0, d.numel(), step):
        a = d[s:s + step].abs()
        if s <= index < s + step:
            a[index - s] = 0
        worst = max(worst, float(a.max()))
    return worst


@pytest.mark.parametrize("name,limit,dtype", [("c3", 12, "complex128"), ("c4", 12, "complex128"),
                                              ("c5_33", 14, "complex128"), ("c3", 12, "complex64")])
def test_full_size_circuit_then_inverse_returns_to_basis(name, limit, dtype):
    """BASELINE configs at their full size (30 / 33 / 33 qubits: 16 / 128 /
    128 GiB, the last two in place) run forward and back through the engine's
    planned passes: the state must return to |0..0> within 1e-10 (complex64:
    1e-4)."""
    c = _inverse_appended(configs.build(name))
    part = partition_dfs(build_dag(c), limit)
    st = execute_hierarchical(c, part, dtype=dtype)
    torch.cuda.synchronize()
    assert _basis_error(st, 0) < TOL[dtype]


def test_bv30_known_answer():
    """30-qubit Bernstein-Vazirani (secret on the odd data qubits 1..27,
    ancilla 29 prepared in |->): the final state is exactly
    (|s> - |s + 2^29>) / sqrt(2) with s = 0xAAAAAAA, a 16 GiB known answer
    that needs no CPU oracle."""
    from paper_2205_06973_b200.qasm import Circuit

    n, anc, s = 30, 29, 0xAAAAAAA
    ops = [GateOp(GateKind.X, (anc,), ())] + [GateOp(GateKind.H, (q,), ()) for q in range(n)]
    ops += [GateOp(GateKind.CX, (q, anc), ()) for q in range(anc) if s >> q & 1]
    ops += [GateOp(GateKind.H, (q,), ()) for q in range(anc)]
    c = Circuit(n, tuple(ops))
    for strategy in (partition_dfs, partition_nat):
        st = execute_hierarchical(c, strategy(build_dag(c), 12))
        d = st.data
        r = 2 ** -0.5
        assert abs(complex(d[s].item()) - r) < 1e-12 and abs(complex(d[s + (1 << anc)].item()) + r) < 1e-12
        d[s] = 0
        d[s + (1 << anc)] = 0
        assert float(d.abs().max()) < 1e-12


@pytest.mark.parametrize("w", [9, 13, 14])
def test_part_apply_c_abi_runs_every_launch(w):
    """hs_part_apply (the C ABI's run_part) on parts whose plan takes
    several launches (w = 13 / 14: tile-sized sub-passes; LAYOUT adds
    restore launches, PINGPONG out-of-place launches, JIT defers the part's
    scalar to the last launch), compared with the oracle's run_part on a
    random batched state."""
    import ctypes

    from paper_2205_06973_b200.hier import _pack

    n, rows = 17, 2
    c = configs.build("c2@17")
    part = partition_dfs(build_dag(c), w).parts[0]
    exe = remap_part(c, part)
    assert exe.num_slots == w
    rng = np.random.default_rng(w)
    data = rng.normal(size=(rows, 1 << n)) + 1j * rng.normal(size=(rows, 1 << n))
    want = data.copy()
    orc.run_part(want, exe.slot_map.qubits, exe.ops, exe.op_slots)
    lib = _native.load()
    eng = _native.engine(0)
    _, gates, total = _pack([exe])
    st = (ctypes.c_int32 * w)(*exe.slot_map.qubits)
    base = _native.HS_PLAN_DEFAULT
    J, L = _native.HS_PLAN_JIT, _native.HS_PLAN_LAYOUT
    for opts in (base, base | L, base | J, base | J | L, base | J | L | _native.HS_PLAN_PINGPONG,
                 base | J | L | _native.HS_PLAN_INIT_LAYOUT | _native.HS_PLAN_NO_RESTORE):
        dev = torch.from_numpy(data.copy()).cuda()
        s = torch.cuda.current_stream().cuda_stream
        _native.check(lib.hs_engine_set_options(eng, opts))
        try:
            _native.check(lib.hs_part_apply(eng, dev.data_ptr(), rows, n, 0, st, w, gates, total, s))
        finally:
            lib.hs_engine_set_options(eng, _native.default_options())
        assert float(np.max(np.abs(dev.cpu().numpy() - want))) < 1e-10, hex(opts)


def test_trace_timing_rows_sum_to_the_program_time():
    """with_timing: every part row carries time_s / hbm_bytes / gbps from
    per-launch CUDA events; the rows add up to the graph-launched program's
    device time within 5 % (the bench's step)."""
    c = configs.build("c2")
    part = partition_dfs(build_dag(c), 12)
    st, tr = execute_hierarchical(c, part, with_trace=True, with_timing=True)
    rows = tr.part_rows()
    assert len(rows) == part.num_parts and all("gbps" in r for r in rows)
    total = sum(r["time_s"] for r in rows)
    run = HierarchicalRun(c, part, basis_start=True)
    from paper_2205_06973_b200.statevec import allocate

    buf = allocate(c.num_qubits)
    for _ in range(3):
        run.program.init_basis(buf, 0)
        run.program.run_graph(buf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(5):
        run.program.init_basis(buf, 0)
        e0.record()
        run.program.run_graph(buf)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    graph_s = sorted(ms)[2] / 1e3
    assert abs(total - graph_s) < 0.05 * graph_s, (total, graph_s)
    assert sum(r["hbm_bytes"] for r in rows) == run.program.num_launches * 2 * (1 << 26) * 16
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    assert max_abs_diff(st, ref) < 1e-10
    # multilevel rows: every level-2 row (or lone level-1 row) is timed
    ml = partition_multilevel(build_dag(configs.build("c2@20")), 12, 8)
    c20 = configs.build("c2@20")
    st, tr = execute_multilevel(c20, ml, with_trace=True, with_timing=True)
    timed = [r for r in tr.part_rows() if "time_s" in r]
    assert timed and sum(r["hbm_bytes"] for r in timed) > 0


def test_distributed_switch_times():
    c = configs.build("c1@16")
    part = partition_dfs(build_dag(c), 8)
    run = simulate_distributed(c, part, 2, with_timing=True)
    stats = run.stats
    assert stats.num_switches > 0 and len(stats.switch_time_s) == stats.num_switches
    doc = stats.to_json()
    assert all(s["time_s"] > 0 for s in doc["switches"]) and doc["totals"]["switch_time_s"] > 0


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_benched_programs_match_c_oracle_at_full_size(name):
    """The exact programs bench.py times, at BASELINE size (c2: 26 qubits,
    c3: 30 qubits, 16 GiB), against the multi-threaded C oracle run on the
    box's host over the same partition (c3: ~70 s on 16 cores) at 1e-10:
    the timed program (|0..0> prepared in its own initial layout, ping-pong
    passes, one CUDA graph launch), the e2e program (natural-order input,
    run_stream from pinned host memory) and the one-pass-per-part program."""
    from paper_2205_06973_b200.statevec import allocate

    c = configs.build(name)
    n = c.num_qubits
    part = partition_dfs(build_dag(c), 12)
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    ref_dev = torch.from_numpy(ref).cuda()
    del ref

    def err(buf):
        from paper_2205_06973_b200.statevec import StateVector

        return max_abs_diff(StateVector(n, buf), ref_dev)

    buf = allocate(n)
    timed = HierarchicalRun(c, part, basis_start=True)
    assert timed.program.initial_layout != tuple(range(n)) and timed.program.needs_scratch
    assert all(timed.program.info(j)["compiled"] for j in range(timed.program.num_launches))
    for _ in range(2):  # graph capture, then replay
        timed.program.init_basis(buf, 0)
        timed.program.run_graph(buf)
        assert err(buf) < 1e-10
    literal = HierarchicalRun(c, part, basis_start=True, options=(timed.program.options & ~_native.HS_PLAN_MERGE)
                              | _native.HS_PLAN_PART_LOCAL)
    assert [literal.program.info(j)["user_part"] for j in range(part.num_parts)] == list(range(part.num_parts))
    literal.program.share_scratch(timed.program._scratch)
    literal.program.init_basis(buf, 0)
    literal.program.run_graph(buf)
    assert err(buf) < 1e-10
    e2e = HierarchicalRun(c, part, basis_start=False)
    e2e.program.share_scratch(timed.program._scratch)
    host_in = torch.zeros(1 << n, dtype=torch.complex128).pin_memory()
    host_in[0] = 1.0
    host_out = torch.empty(1 << n, dtype=torch.complex128).pin_memory()
    e2e.run_stream([host_in, host_in], [host_out, host_out], buffers=[buf])
    torch.cuda.synchronize()
    buf.copy_(host_out)
    assert err(buf) < 1e-10


@pytest.mark.parametrize("policy", ["reference", "lookahead"])
def test_group_run_peer_switches_on_one_gpu(golden, policy):
    """GroupRun: the C multi-device engine (hs_group_switch: pack into
    staging, pull over peer memory with hs_unpack_segments_range_from,
    event-ordered across shard streams) with every shard on device 0, on the
    corpus against the reference's distributed results, and at 24 qubits
    over 4 shards with a small staging buffer (many double-buffered chunks)
    against the C oracle, with per-switch device times."""
    from paper_2205_06973_b200.multi import GroupRun, shard_positions

    docs, states = golden.json("corpus"), golden.npz("corpus")
    checked = 0
    for i, doc in enumerate(docs):
        c = parse_qasm(doc["qasm"])
        for d in doc["dist"]:
            if not d["switches"] or c.num_qubits < 8:
                continue
            R = 1 << d["p"]
            run = GroupRun(c, partition_of(d["parts"]), d["p"], [0] * R, policy=policy, staging_bytes=4096)
            if policy == "reference":
                assert [[list(x.local), list(x.process)] for x in run.layouts] == d["layouts"]
            shards = run.run(run.allocate())
            full = np.zeros(1 << c.num_qubits, dtype=np.complex128)
            for r in range(R):
                full[shard_positions(run.layouts[-1], r)] = shards[r].cpu().numpy()
            assert np.max(np.abs(full - states[f"c{i}"])) < 1e-10, (i, d["p"])
            checked += 1
    assert checked >= 5
    c = configs.build("c3@24")
    part = partition_dfs(build_dag(c), 12)
    run = GroupRun(c, part, 2, [0, 0, 0, 0], policy=policy, staging_bytes=1 << 20)
    assert run.stats.num_switches > 0
    shards = run.run(run.allocate(), with_timing=True)
    assert len(run.stats.switch_time_s) == run.stats.num_switches and min(run.stats.switch_time_s) > 0
    full = np.zeros(1 << c.num_qubits, dtype=np.complex128)
    for r in range(4):
        full[shard_positions(run.layouts[-1], r)] = shards[r].cpu().numpy()
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    assert float(np.max(np.abs(full - ref))) < 1e-10


def test_c_host_program_runs_a_sharded_circuit(tmp_path):
    """A C program (no Python) runs 12 qubits over 2 shards through the C ABI:
    part, hs_group_switch over peer memory, part; it checks the shards
    against its own host simulation and exits 0 below 1e-12."""
    import json
    import subprocess

    from test_native_abi import _build_group_demo

    exe = _build_group_demo(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert json.loads(out.stdout.strip().splitlines()[-1])["max_abs_delta"] < 1e-12


def test_bench_two_ranks_share_one_gpu(tmp_path):
    """bench.py's N > 1 path end to end under torchrun with two ranks on this
    one GPU (gloo for the process group; the test-only HISVSIM_BENCH_* switches):
    weak-scaled workload, sharded run, layout switches over peer memory
    (transport p2p), max-over-ranks timing, e2e and the JSON line."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    import socket

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, HISVSIM_BENCH_ONE_DEVICE="1", HISVSIM_BENCH_BACKEND="gloo",
               HISVSIM_CACHE_DIR=str(tmp_path / "cubins"))
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(root / "bench.py"), "--gpus", "2",
           "--config", "c2", "--steps", "3", "--warmup", "3"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["config"]["num_qubits"] == 27
    assert line["comm"]["transport"] == "p2p" and line["comm"]["switches"] >= 1
    assert line["comm"]["switch_ms_per_step"] > 0 and line["value"] > 0
    assert line["e2e"]["value"] > 0


@pytest.mark.skipif(__import__("os").environ.get("HISVSIM_BIG_ORACLE") != "1",
                    reason="opt-in: ~10 min and 128 GiB of host RAM (HISVSIM_BIG_ORACLE=1)")
def test_full_size_c5_33_matches_c_oracle():
    """c5's per-GPU share at full size (33 qubits, 128 GiB in place, k = 14:
    wide parts as tile sub-passes + restore launches) against the C oracle on
    the box's host (128 GiB, 16 threads), compared chunk by chunk at 1e-10."""
    c = configs.build("c5_33")
    part = partition_dfs(build_dag(c), 14)
    st = execute_hierarchical(c, part)
    torch.cuda.synchronize()
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    step = 1 << 26
    worst = 0.0
    for s in range(0, ref.size, step):
        chunk = torch.from_numpy(ref[s:s + step]).cuda()
        worst = max(worst, float((st.data[s:s + step] - chunk).abs().max()))
        del chunk
    print(f"c5_33 full-size max |delta| {worst:.3e}")
    assert worst < 1e-10
