"""The C ABI library without a GPU: it loads, exports every symbol the
header declares, and its host-side planner produces device programs whose
emulated execution matches the oracle."""

import re
from pathlib import Path

import numpy as np
import pytest

import program_emulator as emu
from conftest import partition_of, parts_of
from oracle import hisim_oracle as orc
from paper_2205_06973_b200 import _native, build_dag, configs, partition_dfs
from paper_2205_06973_b200.errors import PartTooWideForLayoutError
from paper_2205_06973_b200.hier import remap_part
from paper_2205_06973_b200.qasm import Circuit, GateKind, GateOp, parse_qasm

HEADER = Path(__file__).resolve().parent.parent / "include" / "hisvsim.h"


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.load()
    declared = set(re.findall(r"\b(hs_[a-z_0-9]+)\s*\(", HEADER.read_text()))
    assert declared == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.hs_abi_version() == 1


def _emulate_parts(circuit, parts, tile_bits, dtype=0, rows=1, initial=None, options=1):
    n = circuit.num_qubits
    if initial is None:
        psi = np.zeros((rows, 1 << n), dtype=np.complex128)
        psi[:, 0] = 1.0
    else:
        psi = initial.copy()
    for gates, qubits in parts:
        from paper_2205_06973_b200.partition import Part

        exe = remap_part(circuit, Part(0, tuple(gates), tuple(qubits)))
        launch, prog, _ = emu.plan(_native, n, dtype, tile_bits, exe.slot_map.qubits, exe.ops, exe.op_slots, options)
        emu.emulate(psi, n, launch, prog)
    return psi


@pytest.mark.parametrize("tile_bits,options",
                         [(12, 5), (13, 5), (6, 5), (12, 0), (12, 7), (13, 2), (12, 4), (12, 0x15), (10, 0x17)])
def test_planned_programs_match_oracle_on_corpus(golden, tile_bits, options):
    docs, states = golden.json("corpus"), golden.npz("corpus")
    for i, doc in enumerate(docs[:40]):
        c = parse_qasm(doc["qasm"])
        for key, parts in doc["partitions"].items():
            if max(len(q) for _, q in parts) > tile_bits:
                continue
            got = _emulate_parts(c, parts_of(parts), tile_bits, options=options)[0]
            assert np.max(np.abs(got - states[f"c{i}"])) < 1e-12, (i, key)


def test_single_qubit_fusion_shrinks_random_circuit_parts():
    c = configs.build("c2@16")
    part = partition_dfs(build_dag(c), 12).parts[0]
    exe = remap_part(c, part)
    _, _, plain = emu.plan(_native, 16, 0, 12, exe.slot_map.qubits, exe.ops, exe.op_slots, options=0)
    _, _, fused = emu.plan(_native, 16, 0, 12, exe.slot_map.qubits, exe.ops, exe.op_slots, options=1)
    assert fused.input_gates == plain.input_gates == len(exe.ops)
    assert fused.dense_gates < plain.dense_gates
    assert fused.diag_gates == plain.diag_gates  # the CZs stay


@pytest.mark.parametrize("name", ["c3@12", "c4@12"])
def test_parity_diagonals_replace_cx_rz_cx(name):
    """QAOA / Ising bonds (CX . RZ . CX) become one parity diagonal each;
    the emulated program still matches the oracle."""
    c = configs.ising_config(12, 3) if name == "c4@12" else configs.build(name)
    part = partition_dfs(build_dag(c), 10)
    for p in part.parts:
        exe = remap_part(c, p)
        _, _, off = emu.plan(_native, 12, 0, 12, exe.slot_map.qubits, exe.ops, exe.op_slots, options=1)
        _, _, on = emu.plan(_native, 12, 0, 12, exe.slot_map.qubits, exe.ops, exe.op_slots, options=5)
        assert on.perm_gates <= off.perm_gates
    cx = sum(op.kind is GateKind.CX for op in c.ops)
    total_on = 0
    for p in part.parts:
        exe = remap_part(c, p)
        total_on += emu.plan(_native, 12, 0, 12, exe.slot_map.qubits, exe.ops, exe.op_slots, options=5)[2].perm_gates
    assert total_on < cx / 4
    got = _emulate_parts(c, [(p.gate_indices, p.qubits) for p in part.parts], 12, options=5)[0]
    assert np.max(np.abs(got - orc.simulate_flat(c))) < 1e-12


def test_planned_programs_with_batch_rows_and_random_state():
    c = configs.build("c2@11")
    part = partition_dfs(build_dag(c), 7)
    rng = np.random.default_rng(4)
    psi = rng.normal(size=(4, 1 << 11)) + 1j * rng.normal(size=(4, 1 << 11))
    got = _emulate_parts(c, [(p.gate_indices, p.qubits) for p in part.parts], 12, rows=4, initial=psi)
    want = psi.copy()
    for p in part.parts:
        orc.run_part(want, *orc.part_slots(c, p.gate_indices, p.qubits))
    assert np.max(np.abs(got - want)) < 1e-12


def test_swaps_are_relabelled_not_moved():
    c = configs.build("c1@8")
    ops = tuple(range(c.num_ops))
    from paper_2205_06973_b200.partition import Part

    exe = remap_part(c, Part(0, ops, tuple(range(8))))
    launch, prog, info = emu.plan(_native, 8, 0, 12, exe.slot_map.qubits, exe.ops, exe.op_slots)
    assert info.swaps_relabelled == 4
    assert launch["fin_sync"] == 1
    psi = np.zeros((1, 256), dtype=np.complex128)
    psi[0, 0] = 1
    emu.emulate(psi, 8, launch, prog)
    assert np.max(np.abs(psi[0] - orc.simulate_flat(c))) < 1e-12


def test_planner_rejects_bad_parts():
    c = Circuit(14, tuple(GateOp(GateKind.H, (q,)) for q in range(14)))
    from paper_2205_06973_b200.partition import Part

    exe = remap_part(c, Part(0, tuple(range(14)), tuple(range(14))))
    with pytest.raises(PartTooWideForLayoutError):
        emu.plan(_native, 14, 0, 12, exe.slot_map.qubits, exe.ops, exe.op_slots)
    with pytest.raises(ValueError):
        emu.plan(_native, 4, 0, 12, (5,), (GateOp(GateKind.H, (0,)),), ((0,),))
    with pytest.raises(ValueError):
        emu.plan(_native, 4, 0, 12, (2, 1), (GateOp(GateKind.H, (0,)),), ((0,),))


def test_plan_summary_counts():
    c = configs.build("c3@12")
    part = partition_dfs(build_dag(c), 10).parts[1]
    exe = remap_part(c, part)
    _, prog, info = emu.plan(_native, 12, 0, 12, exe.slot_map.qubits, exe.ops, exe.op_slots, options=0)
    kinds = [op.kind for op in exe.ops]
    assert info.input_gates == len(kinds)
    assert info.dense_gates == sum(k in (GateKind.H, GateKind.RX) for k in kinds)
    assert info.perm_gates == kinds.count(GateKind.CX)
    assert info.diag_gates == kinds.count(GateKind.RZ)
    assert info.phases == sum(int(i["op"]) == emu.I_PHASE for i in prog)
    assert info.tile_bits == 12 and info.reg_bits == 4


@pytest.mark.parametrize("name,limit", [("c2@13", 8), ("c3@14", 9), ("c1@12", 6)])
def test_program_layout_and_restore_match_oracle(name, limit):
    """HS_PLAN_LAYOUT: parts permute qubits inside their tiles toward the low
    physical bits, restore launches bring the buffer home; the emulated
    launch sequence must equal the oracle and end in natural order."""
    c = configs.build(name)
    part = partition_dfs(build_dag(c), limit)
    exes = [remap_part(c, p) for p in part.parts]
    want = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in part.parts])
    for tile_bits in (limit, 12):
        launches = emu.plan_program(_native, c.num_qubits, 0, tile_bits, exes, options=5 | 8)
        assert len(launches) >= len(exes)
        psi = np.zeros((1, 1 << c.num_qubits), dtype=np.complex128)
        psi[0, 0] = 1
        for launch, prog in launches:
            emu.emulate(psi, c.num_qubits, launch, prog)
        assert np.max(np.abs(psi[0] - want)) < 1e-12
    # the layout moves at least some later tiles onto the low physical bits
    low = [int(l["tpos"][0]) for l, _ in emu.plan_program(_native, c.num_qubits, 0, 12, exes, options=5 | 8)]
    plain = [int(l["tpos"][0]) for l, _ in emu.plan_program(_native, c.num_qubits, 0, 12, exes, options=5)]
    assert sum(x == 0 for x in low) >= sum(x == 0 for x in plain)


def _final_run(staged, n, tile_bits):
    """Low natural-order qubits the last ping-pong part covers: its own plus
    the lowest others as the tile's extra bits."""
    cov = set(staged)
    for q in range(n):
        if len(cov) >= max(tile_bits, len(staged)):
            break
        cov.add(q)
    run = 0
    while run in cov:
        run += 1
    return run


@pytest.mark.parametrize("name,limit", [("c2@13", 8), ("c3@14", 9), ("c1@12", 6), ("c2@14", 10), ("c4@13", 6)])
def test_pingpong_programs_match_oracle(name, limit):
    """HS_PLAN_PINGPONG: parts alternate state -> scratch -> state, each
    writing the next part's qubits onto the lowest positions; the last part
    writes natural order into the state (no restore launches). Odd and even
    part counts, several tile widths."""
    c = configs.build(name)
    part = partition_dfs(build_dag(c), limit)
    exes = [remap_part(c, p) for p in part.parts]
    want = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in part.parts])
    for tile_bits in (limit, limit + 1, 12):
        launches = emu.plan_program(_native, c.num_qubits, 0, tile_bits, exes, options=5 | 8 | 0x40)
        # at most one gate-free permutation launch at the end (when the last
        # part does not stage all of the planner's `hot` lowest positions)
        hot = min(3, max(1, min(c.num_qubits, tile_bits // 2)))  # final natural-order write: 128 B runs
        assert len(launches) - len(exes) == int(_final_run(part.parts[-1].qubits, c.num_qubits, tile_bits) < hot)
        assert int(launches[-1][0]["out_buf"]) == 0
        oop = [int(l["oop"]) for l, _ in launches]
        assert oop[0] == (len(launches) % 2 == 0) and all(oop[1:])
        psi = np.zeros((1, 1 << c.num_qubits), dtype=np.complex128)
        psi[0, 0] = 1
        emu.run_program(psi, c.num_qubits, launches)
        assert np.max(np.abs(psi[0] - want)) < 1e-12, tile_bits
    # every part after the first reads 128 B runs when the parts overlap enough
    launches = emu.plan_program(_native, c.num_qubits, 0, 12, exes, options=5 | 8 | 0x40)
    low = [sum(int(l["tpos"][b]) == b for b in range(3)) for l, _ in launches[1:]]
    assert sum(x == 3 for x in low) >= len(low) // 2


def _jit_source(c, p, dtype=0, options=5, tile_bits=12):
    import ctypes

    from paper_2205_06973_b200.hier import _pack

    exe = remap_part(c, p)
    _, gates, total = _pack([exe])
    st = (ctypes.c_int32 * max(1, exe.num_slots))(*exe.slot_map.qubits)
    lib = _native.load()
    n = ctypes.c_size_t()
    _native.check(lib.hs_jit_source(c.num_qubits, dtype, tile_bits, options, st, exe.num_slots, gates, total, None, 0,
                                     ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _native.check(lib.hs_jit_source(c.num_qubits, dtype, tile_bits, options, st, exe.num_slots, gates, total, buf,
                                    n.value, ctypes.byref(n)))
    return buf.value.decode()


@pytest.mark.parametrize("name,dtype", [("c2@16", 0), ("c3@16", 0), ("c1@14", 0), ("c2@16", 1)])
def test_compiled_part_sources_build_for_sm100a(tmp_path, name, dtype):
    """The HS_PLAN_JIT code generator emits CUDA that nvcc compiles for
    sm_100a without local-memory spills (NVRTC does the same at run time)."""
    import shutil
    import subprocess

    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    c = configs.build(name)
    part = partition_dfs(build_dag(c), 10)
    for i, p in enumerate(part.parts[:2]):
        src = tmp_path / f"p{i}.cu"
        src.write_text(_jit_source(c, p, dtype))
        res = subprocess.run([nvcc, "-arch=sm_100a", "-cubin", "-o", str(tmp_path / f"p{i}.cubin"), str(src),
                              "-Xptxas", "-v"], capture_output=True, text=True)
        assert res.returncode == 0, res.stderr[-2000:]
        assert "hs_jit_part" in res.stderr


def test_compiled_parts_reconverge_after_tile_waits(tmp_path, monkeypatch):
    """The tile's wait loops are followed by __syncwarp(): without it ptxas
    compiles the rest of the tile as divergent code and keeps the gate
    constants in vector registers, so most DFMAs read three vector operands
    (~2/3 of the DFMA issue rate). With it, the constants sit in uniform
    registers (checked in the SASS: fewer three-vector DFMAs, more UR ones)."""
    import shutil
    import subprocess

    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    c = configs.build("c2@16")
    p = partition_dfs(build_dag(c), 12).parts[0]

    def sass_counts(src):
        (tmp_path / "k.cu").write_text(src)
        res = subprocess.run([nvcc, "-arch=sm_100a", "-cubin", "-o", str(tmp_path / "k.cubin"), str(tmp_path / "k.cu")],
                             capture_output=True, text=True)
        assert res.returncode == 0, res.stderr[-2000:]
        sass = subprocess.run([cuobjdump, "-sass", str(tmp_path / "k.cubin")], capture_output=True, text=True).stdout
        three = ur = 0
        for m in re.finditer(r"\bDFMA\S*\s+([^;]*);", sass):
            srcs = [a.strip() for a in m.group(1).split(",")][1:]
            ur += any("UR" in a for a in srcs)
            three += sum(bool(re.match(r"-?\|?R\d+", a)) for a in srcs) == 3
        return three, ur

    src = _jit_source(c, p)
    wait = src.index("mbarrier.try_wait.parity.shared::cta.b64")
    assert src[wait:].split("\n", 2)[1].strip() == "__syncwarp();"
    three, ur = sass_counts(src)
    monkeypatch.setenv("HISVSIM_SYNCWARP", "0")
    src0 = _jit_source(c, p)
    assert "__syncwarp();" not in src0
    three0, ur0 = sass_counts(src0)
    assert three < three0 and ur > ur0, (three, three0, ur, ur0)


def _structure(m, allow_scale=True):
    import ctypes

    D8 = ctypes.c_double * 8
    a = D8(*np.asarray([[z.real, z.imag] for z in np.asarray(m).ravel()]).ravel())
    s_out, m_out = (ctypes.c_double * 2)(), D8()
    cost = _native.load().hs_structure_2x2(a, int(allow_scale), s_out, m_out)
    mm = np.array([complex(m_out[2 * k], m_out[2 * k + 1]) for k in range(4)]).reshape(2, 2)
    return complex(s_out[0], s_out[1]), mm, cost


def test_structured_2x2_factorisation():
    """Compiled kernels apply M as s * M' with M' snapped to 0/+-1 entries:
    s * M' must equal M to rounding, and the c2/c4 gate set must get cheap."""
    from paper_2205_06973_b200.statevec import gate_matrix

    rng = np.random.default_rng(7)
    cases = {
        "sqrtX": (gate_matrix(GateKind.U3, (np.pi / 2, -np.pi / 2, np.pi / 2)), 4),
        "sqrtY": (gate_matrix(GateKind.U3, (np.pi / 2, 0.0, 0.0)), 4),
        "sqrtW": (gate_matrix(GateKind.U3, (np.pi / 2, -np.pi / 4, np.pi / 4)), 8),
        "H": (gate_matrix(GateKind.H, ()), 4),
        "RX": (gate_matrix(GateKind.RX, (0.37,)), 4),
        "X": (gate_matrix(GateKind.X, ()), 0),
        "Y": (gate_matrix(GateKind.Y, ()), 0),
    }
    for name, (m, want) in cases.items():
        s, mm, cost = _structure(m)
        assert np.max(np.abs(s * mm - m)) < 1e-15, name
        assert cost == want, (name, cost)
    for _ in range(200):
        th, ph, la = rng.uniform(0, 2 * np.pi, 3)
        m = gate_matrix(GateKind.U3, (th, ph, la)) * np.exp(1j * rng.uniform(0, 2 * np.pi))
        s, mm, cost = _structure(m)
        assert np.max(np.abs(s * mm - m)) < 1e-14
        assert cost <= 12  # one entry normalised to 1: 2+2+4+4
        s0, mm0, cost0 = _structure(m, allow_scale=False)
        assert s0 == 1 and cost0 <= 16 and np.max(np.abs(mm0 - m)) < 1e-15


@pytest.mark.parametrize("name,limit,dtype", [("c2@16", 14, 0), ("c2@15", 13, 0), ("c2@17", 14, 1)])
def test_cluster_tile_parts(tmp_path, name, limit, dtype):
    """Parts wider than one CTA's tile (c5's k = 14: 256 KB of complex128)
    are planned as cluster tiles for compiled kernels: the emulated program
    matches the oracle (ping-pong included), the interpreter refuses them,
    and the generated cluster kernel compiles for sm_100a."""
    import shutil
    import subprocess

    c = configs.build(name)
    part = partition_dfs(build_dag(c), limit)
    assert max(len(p.qubits) for p in part.parts) == limit
    exes = [remap_part(c, p) for p in part.parts]
    tile = 12  # compiled programs use 12-bit tiles for both dtypes
    want = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in part.parts])
    for opts in (0x95, 0x95 | 8 | 0x40):  # cluster tiles (HS_PLAN_CLUSTER)
        launches = emu.plan_program(_native, c.num_qubits, dtype, tile, exes, options=opts)
        assert max(int(l["cluster_log"]) for l, _ in launches) == limit - tile
        psi = np.zeros((1, 1 << c.num_qubits), dtype=np.complex128)
        psi[0, 0] = 1
        emu.run_program(psi, c.num_qubits, launches)
        assert np.max(np.abs(psi[0] - want)) < 1e-12
    for opts in (0x5, 0x15, 0x15 | 8 | 0x40):  # default: sub-passes that fit the tile
        launches = emu.plan_program(_native, c.num_qubits, dtype, tile, exes, options=opts)
        assert max(int(l["cluster_log"]) for l, _ in launches) == 0
        assert max(int(l["T"]) for l, _ in launches) <= tile
        assert sum(1 for l, _ in launches) >= len(exes)  # sub-passes (regrouped across parts)
        psi = np.zeros((1, 1 << c.num_qubits), dtype=np.complex128)
        psi[0, 0] = 1
        emu.run_program(psi, c.num_qubits, launches)
        assert np.max(np.abs(psi[0] - want)) < 1e-12
    wide = next(p for p in part.parts if len(p.qubits) == limit)
    src = tmp_path / "cl.cu"
    src.write_text(_jit_source(c, wide, dtype, options=0x95, tile_bits=tile))
    assert "barrier.cluster" in src.read_text()
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    res = subprocess.run([nvcc, "-arch=sm_100a", "-cubin", "-o", str(tmp_path / "cl.cubin"), str(src), "-Xptxas", "-v"],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-3000:]
    spill = int(re.search(r"(\d+) bytes spill stores", res.stderr).group(1))
    assert spill <= 160, res.stderr  # per-tile addresses, outside the gate code


@pytest.mark.parametrize("name,limit,tile", [("c2@16", 14, 12), ("c2@15", 13, 12), ("c4@14", 8, 10), ("c1@13", 6, 10)])
def test_regrouped_passes_match_oracle(name, limit, tile):
    """Wide parts regroup the whole gate stream into tile-sized passes (a pass
    may end one part and start the next; default) unless HS_PLAN_PART_LOCAL;
    HS_PLAN_MERGE regroups even parts that fit. Fewer or equal launches than
    the per-part split, same amplitudes, in place and ping-pong."""
    c = configs.build(name)
    part = partition_dfs(build_dag(c), limit)
    exes = [remap_part(c, p) for p in part.parts]
    want = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in part.parts])
    extra = 0x400 if limit <= tile else 0  # HS_PLAN_MERGE for parts that fit
    for layout in (0, 8, 8 | 0x40):
        local = emu.plan_program(_native, c.num_qubits, 0, tile, exes, options=5 | layout | 0x200)
        merged = emu.plan_program(_native, c.num_qubits, 0, tile, exes, options=5 | layout | extra)
        if layout == 0:  # no restore launches: one launch per pass
            assert len(merged) <= len(local)
            if limit <= tile:
                assert len(local) == len(exes) and len(merged) < len(exes)
        for launches in (local, merged):
            psi = np.zeros((1, 1 << c.num_qubits), dtype=np.complex128)
            psi[0, 0] = 1
            emu.run_program(psi, c.num_qubits, launches)
            assert np.max(np.abs(psi[0] - want)) < 1e-12, (layout, len(launches))


@pytest.mark.parametrize("options", [0x405, 0x40d, 0x44d, 0x415, 0x45d, 0xc15, 0xc5d])
def test_merged_programs_match_oracle_on_corpus(golden, options):
    """Whole programs with HS_PLAN_MERGE (every pass grouping candidate is
    planned and the fewest launches win) on the corpus: tiny states (n < 6,
    where seeds must stay inside the state), every gate kind, with and
    without layouts / ping-pong, with and without global diagonals
    (0x800 with HS_PLAN_JIT), emulated against the reference states."""
    docs, states = golden.json("corpus"), golden.npz("corpus")
    checked = 0
    for i, doc in enumerate(docs[:40]):
        c = parse_qasm(doc["qasm"])
        for key, parts in doc["partitions"].items():
            part = partition_of(parts)
            exes = [remap_part(c, p) for p in part.parts]
            tile = 12
            if max(e.num_slots for e in exes) > tile:
                continue
            launches = emu.plan_program(_native, c.num_qubits, 0, tile, exes, options=options)
            psi = np.zeros((1, 1 << c.num_qubits), dtype=np.complex128)
            psi[0, 0] = 1
            emu.run_program(psi, c.num_qubits, launches)
            assert np.max(np.abs(psi[0] - states[f"c{i}"])) < 1e-12, (i, key)
            checked += 1
    assert checked >= 40


@pytest.mark.parametrize("name,limit", [("c2@20", 12), ("c3@16", 9), ("c1@14", 6), ("c4@13", 6)])
def test_final_layout_is_natural_unless_no_restore(name, limit):
    """hs_program_final_layout's contract: the identity whenever
    HS_PLAN_NO_RESTORE is off, for in-place and ping-pong programs alike
    (including a ping-pong program that ends in a gate-free permutation
    launch); with it on, the layout the emulated program actually left."""
    c = configs.build(name)
    n = c.num_qubits
    exes = [remap_part(c, p) for p in partition_dfs(build_dag(c), limit).parts]
    base = 5 | 0x8  # FUSE_1Q | PARITY | LAYOUT
    for extra in (0, 0x40, 0x40 | 0x400, 0x20, 0x20 | 0x40):
        ip, fp, nl = emu.program_layouts(_native, n, 0, 12, exes, base | extra)
        assert fp == tuple(range(n)), (extra, fp)
        assert nl == len(emu.plan_program(_native, n, 0, 12, exes, base | extra))
    # a 2-part ping-pong program whose last part misses the low positions:
    # the restore launch writes natural order, and the final layout says so
    from paper_2205_06973_b200.partition import Part

    ops = [GateOp(GateKind.H, (q,), ()) for q in range(20)]
    cc = Circuit(20, tuple(ops))
    two = [remap_part(cc, Part(0, tuple(range(0, 12)), tuple(range(0, 12)))),
           remap_part(cc, Part(1, tuple(range(12, 20)), tuple(range(8, 20))))]
    ip, fp, nl = emu.program_layouts(_native, 20, 0, 12, two, base | 0x40)
    assert nl == 3 and fp == tuple(range(20))
    # NO_RESTORE: the reported layout is where the emulated amplitudes are
    ip, fp, nl = emu.program_layouts(_native, n, 0, 12, exes, base | 0x100)
    launches = emu.plan_program(_native, n, 0, 12, exes, base | 0x100)
    psi = np.zeros((1, 1 << n), dtype=np.complex128)
    psi[0, 0] = 1
    emu.run_program(psi, n, launches)
    want = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in partition_dfs(build_dag(c), limit).parts])
    idx = np.arange(1 << n, dtype=np.int64)
    where = np.zeros_like(idx)
    for q in range(n):
        where |= ((idx >> q) & 1) << fp[q]
    assert np.max(np.abs(psi[0][where] - want)) < 1e-12


def _build_group_demo(tmp_path):
    import shutil
    import subprocess

    root = Path(__file__).resolve().parent.parent
    lib = root / "paper_2205_06973_b200" / "_lib"
    exe = tmp_path / "group_demo"
    cc = shutil.which("gcc") or "gcc"
    cmd = [cc, "-O2", "-std=c11", "-I", str(root / "include"), "-I", "/usr/local/cuda/include",
           str(root / "tests" / "c" / "group_demo.c"), "-L", str(lib), "-lhisvsim", "-L", "/usr/local/cuda/lib64",
           "-lcudart", "-lm", f"-Wl,-rpath,{lib}", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_host_program_builds_against_the_header(tmp_path):
    """tests/c/group_demo.c drives a sharded run (programs, hs_group_switch)
    through include/hisvsim.h alone: it compiles and links with gcc."""
    assert _build_group_demo(tmp_path).exists()


def test_grouping_cache_reuses_the_chosen_passes(tmp_path, monkeypatch):
    """The chosen tile-pass grouping is cached on disk: a second plan of the
    same program finds it and emits identical launches; a damaged entry is
    ignored (planned again)."""
    import os
    import subprocess
    import sys

    root = Path(__file__).resolve().parent.parent
    code = ("import sys; sys.path[:0] = [%r, %r]\n"
            "import program_emulator as emu, hashlib\n"
            "from paper_2205_06973_b200 import _native, build_dag, configs, partition_dfs\n"
            "from paper_2205_06973_b200.hier import remap_part\n"
            "c = configs.build('c3@20'); ex = [remap_part(c, p) for p in partition_dfs(build_dag(c), 9).parts]\n"
            "L = emu.plan_program(_native, 20, 0, 12, ex, 0x47d | 0x8 | 0x20)\n"
            "print(len(L), hashlib.sha1(b''.join(l.tobytes() + p.tobytes() for l, p in L)).hexdigest())\n"
            % (str(root), str(root / "tests")))
    env = dict(os.environ, HISVSIM_CACHE_DIR=str(tmp_path))
    first = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True).stdout
    files = list(tmp_path.glob("*.grouping"))
    assert len(files) == 1
    second = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True).stdout
    assert first == second
    files[0].write_bytes(b"garbage")
    third = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True).stdout
    assert third == first


@pytest.mark.parametrize("name,limit,tile", [("c3@16", 8, 10), ("c4@15", 8, 10), ("c2@16", 8, 10), ("c3@14", 6, 8),
                                             ("c1@13", 6, 10)])
def test_global_diagonal_programs_match_oracle(name, limit, tile, monkeypatch):
    """HS_PLAN_GLOBAL_DIAG: regrouped passes stage only the qubits their
    non-diagonal gates act on; diagonal gates (CZ, parity diagonals of
    CX.RZ.CX, Z-type gates) on unstaged qubits read those qubits' values from
    the tile's free index bits (I_GLOBALS + the gq / gc masks of DIAG
    instructions). Fewer launches than the staged-diagonal grouping, the
    same amplitudes, in place and ping-pong, emulated against the oracle
    (HISVSIM_GLOBAL_DIAG=1: also for circuits below the diagonal share the
    planner asks for by default)."""
    monkeypatch.setenv("HISVSIM_GLOBAL_DIAG", "1")
    c = configs.build(name)
    part = partition_dfs(build_dag(c), limit)
    exes = [remap_part(c, p) for p in part.parts]
    want = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in part.parts])
    with_globals = 0
    for layout in (0, 8, 8 | 0x40):
        staged = emu.plan_program(_native, c.num_qubits, 0, tile, exes, options=0x415 | layout)
        glob = emu.plan_program(_native, c.num_qubits, 0, tile, exes, options=0xc15 | layout)
        assert len(glob) <= len(staged)
        with_globals += sum(1 for _, prog in glob if len(prog) and int(prog[0]["op"]) == emu.I_GLOBALS)
        for launches in (staged, glob):
            psi = np.zeros((1, 1 << c.num_qubits), dtype=np.complex128)
            psi[0, 0] = 1
            emu.run_program(psi, c.num_qubits, launches)
            assert np.max(np.abs(psi[0] - want)) < 1e-12, (layout, len(launches))
    if not name.startswith("c1"):
        assert with_globals > 0


def test_global_diagonals_cut_the_c3_and_c4_launch_counts():
    """The BASELINE configs' full-size programs (planning is host-only):
    c3 (30-qubit QAOA, k = 12) 13 -> 7 launches, c4 (33-qubit TFIM) 46 -> 27
    with unstaged diagonals; HS_PLAN_GLOBAL_DIAG off keeps the old plans, and
    so do random circuits (c2: CZs are 26 % of the units, below the 40 % the
    planner asks for; measured slower there)."""
    import os

    old = os.environ.get("HISVSIM_CACHE_DIR")
    os.environ["HISVSIM_CACHE_DIR"] = "off"
    try:
        for name, opts, most in (("c3", 0x47d, 8), ("c4", 0x41d, 30)):
            c = configs.build(name)
            part = partition_dfs(build_dag(c), configs.CONFIGS[name].limit)
            exes = [remap_part(c, p) for p in part.parts]
            staged = emu.plan_program(_native, c.num_qubits, 0, 12, exes, options=opts)
            glob = emu.plan_program(_native, c.num_qubits, 0, 12, exes, options=opts | 0x800)
            assert len(glob) <= most < len(staged), (name, len(glob), len(staged))
            assert not any(len(p) and int(p[0]["op"]) == emu.I_GLOBALS for _, p in staged)
        c = configs.build("c2")
        part = partition_dfs(build_dag(c), 12)
        exes = [remap_part(c, p) for p in part.parts]
        plan = emu.plan_program(_native, c.num_qubits, 0, 12, exes, options=0xc7d)
        assert not any(len(p) and int(p[0]["op"]) == emu.I_GLOBALS for _, p in plan)
    finally:
        if old is None:
            os.environ.pop("HISVSIM_CACHE_DIR", None)
        else:
            os.environ["HISVSIM_CACHE_DIR"] = old


def test_global_diagonal_edge_circuits(monkeypatch):
    """Edge cases of unstaged diagonals, emulated against the oracle: a
    circuit of diagonal gates only (passes that stage nothing), a graph
    state (H on every qubit, CZ on every pair: CZs with both qubits global),
    and controlled phases whose control or target is the only unstaged
    qubit; tiles narrower than the state so globals are free bits."""
    import random

    from paper_2205_06973_b200.qasm import Circuit, GateKind, GateOp

    monkeypatch.setenv("HISVSIM_GLOBAL_DIAG", "1")
    rng = random.Random(7)
    n = 13
    diag_only = [GateOp(GateKind.H, (q,), ()) for q in (0, 5)]
    for _ in range(120):
        a, b = rng.sample(range(n), 2)
        k = rng.choice([GateKind.Z, GateKind.S, GateKind.T, GateKind.RZ, GateKind.U1, GateKind.CZ, GateKind.CRZ])
        if k in (GateKind.CZ, GateKind.CRZ):
            diag_only.append(GateOp(k, (a, b), (rng.uniform(0, 3),) if k == GateKind.CRZ else ()))
        else:
            diag_only.append(GateOp(k, (a,), (rng.uniform(0, 3),) if k in (GateKind.RZ, GateKind.U1) else ()))
    graph = [GateOp(GateKind.H, (q,), ()) for q in range(n)]
    graph += [GateOp(GateKind.CZ, (a, b), ()) for a in range(n) for b in range(a + 1, n) if (a * 7 + b) % 3]
    graph += [GateOp(GateKind.RX, (q,), (0.3 + q,)) for q in range(n)]
    ctl = [GateOp(GateKind.H, (q,), ()) for q in range(n)]
    for layer in range(3):
        for q in range(n - 1):
            ctl.append(GateOp(GateKind.CRZ, (q, n - 1 - q) if q != n - 1 - q else (q, 0), (0.1 * (q + layer + 1),)))
        ctl += [GateOp(GateKind.RY, (q,), (0.2 * layer + 0.1,)) for q in range(0, n, 2)]
    for ops in (diag_only, graph, ctl):
        c = Circuit(n, tuple(ops))
        with_globals = 0
        for limit in (4, 6):
            part = partition_dfs(build_dag(c), limit)
            exes = [remap_part(c, p) for p in part.parts]
            want = orc.execute_hierarchical(c, [(p.gate_indices, p.qubits) for p in part.parts])
            for tile, opts in ((6, 0xc15), (8, 0xc1d), (8, 0xc5d)):
                launches = emu.plan_program(_native, n, 0, tile, exes, options=opts)
                psi = np.zeros((1, 1 << n), dtype=np.complex128)
                psi[0, 0] = 1
                emu.run_program(psi, n, launches)
                assert np.max(np.abs(psi[0] - want)) < 1e-12, (limit, tile, hex(opts))
                with_globals += sum(1 for _, p in launches if len(p) and int(p[0]["op"]) == emu.I_GLOBALS)
        assert with_globals > 0
