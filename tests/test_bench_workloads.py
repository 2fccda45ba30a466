"""bench.py's workloads at every GPU count the driver runs (N = 1, 2, 4, 8),
built and planned on the host: the circuit generator accepts the size, the
partition covers it, the sharded run's layout schedule exists, and every
segment program of every rank plans (hs_plan_program_layouts, no GPU)."""

import sys
from pathlib import Path

import pytest

import program_emulator as emu
from paper_2205_06973_b200 import _native, configs
from paper_2205_06973_b200.hier import remap_part

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

EXPECT = {  # config -> {N: (qubits, scaling)}
    "c1": {1: (20, "weak"), 2: (21, "weak"), 4: (22, "weak"), 8: (23, "weak")},
    "c2": {1: (26, "weak"), 2: (27, "weak"), 4: (28, "weak"), 8: (29, "weak")},
    "c3": {1: (30, "weak"), 2: (31, "weak"), 4: (32, "weak"), 8: (33, "weak")},
    "c4": {1: (33, "strong"), 2: (33, "strong"), 4: (33, "strong"), 8: (33, "strong")},
    "c5": {1: (33, "weak"), 2: (34, "weak"), 4: (35, "weak"), 8: (36, "weak")},
}


@pytest.mark.parametrize("config", sorted(EXPECT))
@pytest.mark.parametrize("gpus", [1, 2, 4, 8])
def test_every_bench_workload_builds_and_plans(config, gpus):
    from paper_2205_06973_b200.multi import ShardedRun

    name, scaling = configs.bench_workload(config, gpus)
    n, want_scaling = EXPECT[config][gpus]
    assert scaling == want_scaling
    cfg, circuit, part, _ = bench.build_workload(name, "dfs")
    assert circuit.num_qubits == n
    assert sorted(g for p in part.parts for g in p.gate_indices) == list(range(circuit.num_ops))
    assert max(len(p.qubits) for p in part.parts) <= cfg.limit
    p = gpus.bit_length() - 1
    base = _native.HS_PLAN_DEFAULT | _native.HS_PLAN_LAYOUT
    if p == 0:
        exes_list = [[remap_part(circuit, q) for q in part.parts]]
        n_local = n
    else:
        run = ShardedRun(circuit, part, p, program=False, loopback=True)
        assert run.n_local == n - p
        n_local = run.n_local
        exes_list = []
        for a, b in run.segments:
            if b > a:
                exes_list.append(run.exes[run.bounds[a][0]:run.bounds[b - 1][0] + run.bounds[b - 1][1]])
        assert run.stats.num_switches == len(run.segments) - 1
    for exes in exes_list:
        ip, fp, nl = emu.program_layouts(_native, n_local, 0, 12, exes, base)
        assert nl >= 1 and fp == tuple(range(n_local))


def test_qaoa_odd_sizes_are_near_regular():
    import random

    for n in (31, 33):
        edges = configs.qaoa_graph(n, random.Random(0))
        deg = [0] * n
        for a, b in edges:
            assert 0 <= a < b < n
            deg[a] += 1
            deg[b] += 1
        assert sorted(deg) == [2, 2, 2] + [3] * (n - 3)
    # even sizes keep the exact 3-regular graph (c3 itself is unchanged)
    assert configs.qaoa_graph(30, random.Random(0)) == configs.random_3_regular(30, random.Random(0))


def test_c5_sizes_and_rejections():
    assert [configs.build(f"c5@{n}").num_qubits for n in (33, 34, 35, 36)] == [33, 34, 35, 36]
    assert configs.build("c5@34").ops == configs.build("c5_34").ops
    with pytest.raises(KeyError):
        configs.build("c5_33@30")
    with pytest.raises(KeyError):
        configs.build("c5@32")
    with pytest.raises(ValueError):
        configs.bench_workload("c5", 16)
    with pytest.raises(ValueError):
        configs.bench_workload("c3", 3)


def test_reference_arm_line_counts_the_same_work(tmp_path):
    """`bench.py --impl reference` (the CPU restatement, no GPU) prints the
    contract's JSON line in the engine arm's unit: amplitude updates of the
    reference partition per second (2 x 16 B each), with the sampled bytes
    beside it, so the driver's ratio compares the same work."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    import bench

    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "1", "--cpu-step-seconds", "0.2"],
                         capture_output=True, text=True, timeout=600, cwd=tmp_path)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == bench.UNIT
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert abs(line["hbm_gbs_moved"] - line["value"] * bench.AMP_BYTES_PER_UPDATE) < 1e-6 * line["hbm_gbs_moved"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
