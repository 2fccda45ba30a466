"""The command line (paper_2205_06973_b200.cli): partition JSON, exit-code
contract (0 ok, 1 usage, 2 input, 3 verification); ``run`` on the GPU."""

import json

import numpy as np
import pytest

from paper_2205_06973_b200 import cli


def test_partition_writes_reference_json(tmp_path, capsys):
    out = tmp_path / "p.json"
    assert cli.main(["partition", "c1", "--strategy", "dfs", "--limit", "10", "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["strategy"] == "dfs" and doc["limit"] == 10
    assert len(doc["parts"]) == 17  # c1 dfs at k=10
    dot = tmp_path / "g.dot"
    assert cli.main(["partition", "c2@12", "--strategy", "multilevel", "--l1", "8", "--l2", "4",
                     "--dag", str(dot)]) == 0
    assert dot.read_text().startswith("digraph")


def test_exit_codes(tmp_path):
    assert cli.main(["partition"]) == 1                       # usage: missing circuit
    assert cli.main(["partition", "c1", "--strategy", "bogus"]) == 1
    assert cli.main(["partition", "no_such_circuit"]) == 2    # input
    bad = tmp_path / "bad.qasm"
    bad.write_text("OPENQASM 2.0;\nqreg q[2];\nfoo q[0];\n")
    assert cli.main(["partition", str(bad)]) == 2
    assert cli.main(["partition", "c1", "--limit", "1"]) == 2  # limit below the widest gate


@pytest.mark.gpu
def test_run_hierarchical_report_trace_state(tmp_path, golden):
    rep, tr, st = tmp_path / "r.json", tmp_path / "t.jsonl", tmp_path / "s.bin"
    code = cli.main(["run", "c1@12", "--mode", "hierarchical", "--strategy", "dagp", "--limit", "6", "--verify",
                     "--report", str(rep), "--trace", str(tr), "--out", str(st)])
    assert code == 0
    r = json.loads(rep.read_text())
    assert r["num_parts"] == len(r["parts"]) and r["max_abs_delta"] < 1e-10
    assert len(tr.read_text().strip().splitlines()) == r["num_parts"]
    amps = np.fromfile(st, dtype="<c16")
    assert amps.size == 1 << 12 and abs(np.linalg.norm(amps) - 1) < 1e-12
    assert cli.main(["run", "c1@12", "--mode", "distributed", "--p", "2", "--limit", "6", "--verify"]) == 0
    assert cli.main(["run", "c1@12", "--mode", "multilevel", "--l1", "8", "--l2", "4", "--verify"]) == 0
    assert cli.main(["run", "c1@12", "--mode", "flat", "--trace", str(tr)]) == 1  # usage


@pytest.mark.gpu
def test_verification_failure_is_exit_three(capsys, monkeypatch):
    """The reference's fault injection (tests/test_cli.py:62-79): a
    corrupted executor must fail --verify with exit code 3, which only
    holds because verify compares against the independent gate-by-gate run."""
    from paper_2205_06973_b200 import hier

    real = hier.execute_hierarchical

    def corrupted(circuit, partition, **kwargs):
        out = real(circuit, partition, **kwargs)
        state = out[0] if isinstance(out, tuple) else out
        state.data[0] += 0.5
        return out

    monkeypatch.setattr(hier, "execute_hierarchical", corrupted)
    code = cli.main(["run", "c1@12", "--mode", "hierarchical", "--limit", "6", "--verify"])
    assert code == 3
    assert "delta" in capsys.readouterr().err


@pytest.mark.gpu
def test_verify_runs_one_interpreter_launch_per_gate():
    """verify_against_flat's reference run is the literal gate-by-gate
    program: as many launches as gates, none compiled, natural order."""
    from paper_2205_06973_b200 import build_dag, configs, partition_dfs
    from paper_2205_06973_b200.hier import execute_hierarchical, flat_program, verify_against_flat

    for name in ("c2@20", "c3@20"):
        c = configs.build(name)
        prog = flat_program(c)
        assert prog.num_launches == c.num_ops
        assert prog.initial_layout == prog.final_layout == tuple(range(c.num_qubits))
        assert not any(prog.info(i)["compiled"] for i in range(prog.num_launches))
        st = execute_hierarchical(c, partition_dfs(build_dag(c), 12))
        assert verify_against_flat(c, st) < 1e-10
