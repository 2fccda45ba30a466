"""Benchmark: circuit time-to-solution and effective HBM GB/s per part-pass.

One step = one full simulation of the BASELINE config circuit on a state
already resident in HBM: every tile pass the planner made of the
partition's parts (csrc/hs_planner.cpp group_passes), plus any gate-free
layout launch. ``value`` = the reference's work per circuit - every part of
the partition updates every amplitude once (parts x 2^n amplitude updates,
summed over ranks) - / time-to-solution: the same count on the reference
arm, whatever number of launches the engine groups the parts into.
``hbm_gbs_moved`` = HBM bytes the step's launches actually move (each launch
reads and writes every amplitude of a rank's shard: 2 x 2^l x 16 B) / step
time, never above the HBM peak; ``roofline`` explains it per launch. ``ms_per_step`` is the circuit
time-to-solution; partitioning and planning (host) are reported
separately. ``e2e`` is the same metric through the public API with the
initial state in pinned host memory and the final state read back every
step. ``one_pass_per_part`` times the literal reference granularity (one
pass per part, HS_PLAN_PART_LOCAL, no merging) beside the default.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--strategy dfs]
    python bench.py --impl reference ...   # the CPU port of the reference path

Workloads per N (paper_2205_06973_b200.configs.bench_workload): c1 / c2 /
c3 weak-scale to n + log2 N qubits, c4 is 33 qubits at every N (strong),
c5 is 33 / 34 / 35 / 36 qubits at 1 / 2 / 4 / 8 GPUs. Under torchrun
(N > 1) the state is sharded over the ranks and layout switches run over
NCCL.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "circuit time-to-solution and effective HBM GB/s per part-pass at 1/2/4/8 B200"
#: The reference's unit of work: one part updates every amplitude of the
#: state once (its gather -> gates -> scatter pass, hier.py:220-244).
#: value = parts x 2^n amplitude updates (all ranks) / time-to-solution; it
#: counts the same work on both arms however the engine groups the parts
#: into launches. HBM bytes the launches actually move are reported beside
#: it (hbm_gbs_moved, never above the HBM peak) and in `roofline`.
UNIT = "G part-amplitude updates/s"
AMP_BYTES_PER_UPDATE = 32  # one read + one write of a complex128 amplitude


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def _traffic_from_profiles(config: str, strategy: str):
    """Per-launch DRAM bytes of the part kernel from the committed ncu
    summary of this workload (profiles/*_ncu_summary.json), else None."""
    best = None  # the latest capture: highest capture_seq, else a "final" one
    for f in sorted((ROOT / "profiles").glob("*ncu_summary.json")):
        try:
            d = json.loads(f.read_text())
        except Exception:
            continue
        v = d.get("dram_bytes_per_launch")
        if d.get("workload") == f"{config}/{strategy}" and v and v == v:  # (v == v: not NaN)
            key = (int(d.get("capture_seq", 1 if "final" in f.name else 0)), f.name)
            if best is None or key > best[0]:
                best = (key, float(d["dram_bytes_per_launch"]))
    return best[1] if best else None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm, smax, power = [], [], []
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                power.append(float(r[2]))
            except ValueError:
                continue
            for name, v in zip(names, r[3:7]):
                if v.strip().lower() in ("active", "1"):
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None, "samples": len(sm), "reasons": sorted(reasons)}


def build_workload(name: str, strategy: str, limit: int | None = None, partition_file: str | None = None):
    """Circuit + partition of a bench workload (``configs.bench_workload``'s
    circuit name) and the host partitioning time; ``partition_file``: a
    partition JSON (the reference's document, e.g. from ``cli partition``)."""
    from paper_2205_06973_b200 import build_dag, configs, partition_dagp, partition_dfs, partition_nat
    from paper_2205_06973_b200.partition import partition_from_json

    cfg = configs.CONFIGS[name.split("@")[0]]
    circuit = configs.build(name)
    t0 = time.perf_counter()
    if partition_file:
        part = partition_from_json(build_dag(circuit), Path(partition_file).read_text())
        return cfg, circuit, part, time.perf_counter() - t0
    fn = {"nat": partition_nat, "dfs": partition_dfs, "dagp": partition_dagp}[strategy]
    part = fn(build_dag(circuit), limit or cfg.limit)
    t_part = time.perf_counter() - t0
    return cfg, circuit, part, t_part


# --------------------------------------------------------------------------- CPU reference arm

def cpu_arm(args, cfg, circuit, part, t_part, steps, warmup):
    """The reference path's CPU restatement (oracle/sv_oracle.c, all host
    threads) on a bounded sample of fixings of every part."""
    import numpy as np

    from oracle import c_oracle

    c_oracle.lib()
    threads = c_oracle.threads()
    n = circuit.num_qubits
    slots = [c_oracle.part_slots(circuit, p.gate_indices, p.qubits) for p in part.parts]
    # a state that does not fit the host (36 qubits = 1 TiB) is sampled on a
    # host-sized one: each part keeps its gates, width and the order of its
    # positions, compressed onto the lowest qubits that fit (the sample only
    # sets the lowest free bits of a fixing anyway); said in `sample`
    host = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    n_host = n
    while (16 << n_host) > 0.4 * host and n_host > 1 + max(len(pos) for pos, _, _ in slots):
        n_host -= 1
    if n_host < n:
        squeezed = []
        for pos, ops, sl in slots:
            top = n_host - len(pos)  # keep positions below `top`, move the rest just below n_host
            high = [q for q in pos if q >= top]
            remap = {q: (q if q < top else top + high.index(q)) for q in pos}
            squeezed.append((tuple(sorted(remap[q] for q in pos)), ops, sl))
        slots = squeezed
        n = n_host
    # calibrate: fixings per part so that one step takes ~target seconds
    target = args.cpu_step_seconds
    psi = np.empty(1 << n, dtype=np.complex128)
    psi.fill(0)  # fault the pages in before timing anything
    psi[0] = 1.0
    def make_plan(frac):
        return [(pos, ops, sl, max(1, min(1 << (n - len(pos)), int((1 << (n - len(pos))) * frac))))
                for pos, ops, sl in slots]

    def timed(plan):
        t0 = time.perf_counter()
        for pos, ops, sl, k in plan:
            c_oracle.run_part(psi, pos, ops, sl, 0, k)
        return time.perf_counter() - t0

    frac = 1e-4
    timed(make_plan(frac))
    while True:  # grow the sample until a pass is long enough to time
        dt = timed(make_plan(frac))
        if dt > 0.25 or frac >= 1.0:
            break
        frac = min(1.0, frac * 8)
    frac = min(1.0, frac * target / dt)
    plan = make_plan(frac)

    def step():
        b = 0
        for pos, ops, sl, k in plan:
            c_oracle.run_part(psi, pos, ops, sl, 0, k)
            b += 2 * (k << len(pos)) * 16
        return b

    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    nbytes = 0
    for _ in range(steps):
        nbytes += step()
    dt = time.perf_counter() - t0
    gbs = nbytes / dt / 1e9
    value = gbs / AMP_BYTES_PER_UPDATE  # G amplitude updates / s
    sample_amps = sum(k << len(pos) for pos, _, _, k in plan)
    sample = (("" if n == circuit.num_qubits else
               f"state squeezed to {n} of {circuit.num_qubits} qubits to fit the host (parts' positions "
               f"compressed onto the lowest qubits); ") +
              f"{config_label(args)}: each step runs every one of the {len(plan)} parts over "
              f"{sample_amps / (1 << n) / len(plan):.4%} of its fixings ({sample_amps} amplitude updates "
              f"per step, fixings 0..k-1 of each part) with {threads} threads; value = amplitude updates / "
              f"time, the same count as the GPU arm (gbs = 2 x 16 B per update)")
    full_s = (len(plan) * (1 << n)) / (value * 1e9)
    return {
        "value": value, "gbs": gbs, "threads": threads, "sample": sample, "ms_per_step": dt / steps * 1e3,
        "projected_time_to_solution_s": full_s,
    }


def numpy_port_c1_seconds():
    """The reference's own numpy algorithm (oracle/hisim_oracle.py, a
    restatement of hisim.hier.execute_hierarchical: per part one batched
    fancy-index gather, numpy ufunc gates, scatter) on c1 (20 qubits, dfs,
    k = 10), one core: the reference CPU path's speed at the one BASELINE
    config it runs in seconds (the C port above is the stronger baseline)."""
    from oracle import hisim_oracle as orc
    from paper_2205_06973_b200 import build_dag, configs, partition_dfs

    c = configs.build("c1")
    parts = [(p.gate_indices, p.qubits) for p in partition_dfs(build_dag(c), 10).parts]
    t0 = time.perf_counter()
    orc.execute_hierarchical(c, parts)
    return time.perf_counter() - t0


def config_label(args):
    return f"{args.workload}/{args.strategy}"


# --------------------------------------------------------------------------- GPU arm

def plan_probe(args) -> int:
    """--plan-probe: plan + compile the workload's program in this (fresh)
    process and print the host seconds it took (the disk cubin cache is
    whatever HISVSIM_CACHE_DIR holds)."""
    import torch

    from paper_2205_06973_b200 import _native
    from paper_2205_06973_b200.hier import HierarchicalRun

    _, circuit, part, _ = build_workload(args.workload, args.strategy, args.limit, args.partition)
    torch.cuda.init()
    _native.engine(0)
    t0 = time.perf_counter()
    HierarchicalRun(circuit, part, device="cuda:0", options=args.plan_options, basis_start=True)
    dt = time.perf_counter() - t0
    print(json.dumps({"plan_seconds": dt, "jit": _native.jit_cache_stats()}), flush=True)
    return 0


def _warm_plan_seconds(args):
    """Plan time of the same program in a second process that finds the
    cubins this process compiled in the on-disk cache."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--plan-probe", "--config", args.config, "--strategy",
           args.strategy]
    if args.limit:
        cmd += ["--limit", str(args.limit)]
    if args.plan_options is not None:
        cmd += ["--plan-options", hex(args.plan_options)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ))
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:  # reported, never fatal for the bench line
        return {"error": f"{type(exc).__name__}: {exc}"}


def _time_program(run, state, steps, launch, stream):
    """Device ms per step of ``launch`` over ``steps`` steps, each step's
    basis state prepared outside the timed window (events on the launch
    stream)."""
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for e0, e1 in ev:
        run.program.init_basis(state, 0)
        e0.record(stream)
        launch(state)
        e1.record(stream)
    torch.cuda.synchronize()
    return sum(e0.elapsed_time(e1) for e0, e1 in ev) / steps


def gpu_arm(args, circuit, part, rank, world):
    import torch

    from paper_2205_06973_b200 import _native
    from paper_2205_06973_b200.hier import HierarchicalRun
    from paper_2205_06973_b200.statevec import allocate, init_basis

    # HISVSIM_BENCH_ONE_DEVICE=1 (tests only): every rank on cuda:0, to run the
    # N > 1 path on a one-GPU box with HISVSIM_BENCH_BACKEND=gloo
    local = 0 if os.environ.get("HISVSIM_BENCH_ONE_DEVICE") == "1" else int(os.environ.get("LOCAL_RANK", 0))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    _native.engine(dev.index or 0)
    n = circuit.num_qubits
    dist = world > 1
    # host planning: the planner + NVRTC code generation of every pass
    # (cold: this process's own cubin cache directory starts empty)
    t0 = time.perf_counter()
    if dist:
        from paper_2205_06973_b200.multi import ShardedRun

        # layout switches pull over peer memory (CUDA IPC) when every rank can
        # map its peers' staging, else batched NCCL send/recv
        run = ShardedRun(circuit, part, int(math.log2(world)), device=dev, transport="auto")
        n_local = run.n_local
    else:
        # the timed runs start from |0..0>, prepared in the program's layout
        run = HierarchicalRun(circuit, part, device=dev, options=args.plan_options, basis_start=True)
        n_local = n
    plan_s = time.perf_counter() - t0
    jit_stats = _native.jit_cache_stats()
    num_parts = part.num_parts
    programs = [run.program] if not dist else [pr for pr in run.programs if pr is not None]
    num_launches = sum(pr.num_launches for pr in programs)
    bytes_per_pass = 2 * (1 << n_local) * 16
    launch_owner = [run.program.info(j)["user_part"] for j in range(num_launches)] if not dist else []
    state = allocate(n_local, "complex128", dev)
    stream = torch.cuda.current_stream(dev)

    # the whole program as one CUDA graph launch (PartProgram.run_graph,
    # captured in the warm-up) unless --no-graph: launch overhead matters for
    # L2-resident states (c1: 7 launches of ~16 us)
    def launch(buf, r=run):
        if args.no_graph:
            r.program.run(buf)
        else:
            r.program.run_graph(buf, stream=stream)

    def prepare():
        if not dist:
            run.program.init_basis(state, 0)
        elif rank == 0:
            init_basis(state, 0)
        else:
            state.zero_()

    def one_step(timed_events=None):
        prepare()
        if timed_events is not None:
            timed_events.append(torch.cuda.Event(enable_timing=True))
            timed_events[-1].record(stream)
        if dist:
            marks_ = []
            run.run(state, events=marks_)
            if timed_events is not None:
                timed_events += marks_
        elif timed_events is None:
            launch(state)
        else:
            for i in range(num_launches):
                run.program.run(state, i, 1)
                timed_events.append(torch.cuda.Event(enable_timing=True))
                timed_events[-1].record(stream)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    clocks.start()
    # K timed steps: each step's initial state is prepared first (t_init,
    # reported apart: the input is resident when the hot path starts), then
    # all launches (and switches) run between two events on the launch stream
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for e_init, e0, e1 in step_ev:
        e_init.record(stream)
        prepare()
        e0.record(stream)
        if dist:
            run.run(state)
        else:
            launch(state)
        e1.record(stream)
    torch.cuda.synchronize()
    total_ms = sum(e0.elapsed_time(e1) for _, e0, e1 in step_ev)
    init_ms = sum(ei.elapsed_time(e0) for ei, e0, _ in step_ev) / args.steps
    clk = clocks.stop()
    # per-launch durations (events between launches) from further untimed steps
    marks = []
    for _ in range(min(args.steps, 3)):
        ev = []
        one_step(ev)
        marks.append(ev)
    torch.cuda.synchronize()
    n_marked = len(marks)
    # per launch of the part kernel (events between launches); distributed:
    # per segment ("parts") and per layout switch ("switch")
    durs, restore_ms, seg_ms = [], 0.0, 0.0
    switch_list = []  # ms of each switch, per marked step
    launch_ms = []  # per launch, per marked step
    for ev in marks:
        if dist:
            sw = []
            for i in range(1, len(ev)):
                kind, e = ev[i]
                prev = ev[i - 1][1] if isinstance(ev[i - 1], tuple) else ev[i - 1]
                if kind == "switch":
                    sw.append(prev.elapsed_time(e))
                else:
                    seg_ms += prev.elapsed_time(e)
            switch_list.append(sw)
            continue
        d = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)]
        launch_ms.append(d)
        # a launch belongs to a caller's part (wide parts may take several
        # sub-pass launches) or is a gate-free layout launch (user_part -1)
        per_part = [0.0] * num_parts
        for j, dj in enumerate(d):
            u = launch_owner[j]
            if u >= 0:
                per_part[u] += dj
            else:
                restore_ms += dj
        durs += per_part
    if dist:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    moved = world * num_launches * bytes_per_pass  # HBM bytes of all ranks' launches per step
    hbm_gbs = moved / (ms_step / 1e3) / 1e9
    part_amps = world * num_parts * (1 << n_local)  # the reference's work: every part updates every amplitude
    value = part_amps / (ms_step / 1e3) / 1e9

    # the literal reference granularity: one pass per part (no merging or
    # regrouping of parts into tile passes), same layouts / JIT / graph
    literal = None
    if not dist and not args.no_literal:
        opts = (run.program.options & ~_native.HS_PLAN_MERGE) | _native.HS_PLAN_PART_LOCAL
        lit = HierarchicalRun(circuit, part, device=dev, options=opts, basis_start=True)
        if lit.program.needs_scratch and run.program.needs_scratch:
            lit.program.share_scratch(run.program._scratch)
        for _ in range(max(1, args.warmup)):
            lit.program.init_basis(state, 0)
            launch(state, lit)
        lit_ms = _time_program(lit, state, args.steps, lambda b: launch(b, lit), stream)
        nl = lit.program.num_launches
        literal = {"ms_per_step": lit_ms, "launches_per_step": nl, "parts": num_parts,
                   "value": num_parts * (1 << n_local) / (lit_ms / 1e3) / 1e9, "unit": UNIT,
                   "hbm_gbs_moved": nl * bytes_per_pass / (lit_ms / 1e3) / 1e9,
                   "options": hex(opts),
                   "note": "HS_PLAN_PART_LOCAL without HS_PLAN_MERGE: every launch carries one part's gates "
                           "(plus gate-free layout launches); the default regroups parts into tile passes"}
        del lit

    # e2e through the public API: host initial state in, host state out
    e2e = None
    host_total = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    e2e_fits = world * 2 * ((1 << n_local) * 16) <= 0.4 * host_total and (1 << n_local) * 16 <= E2E_MAX_STATE_BYTES
    if dist and not args.no_e2e and not e2e_fits:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "skipped": f"{world} ranks x 2 pinned host buffers of a {((1 << n_local) * 16) >> 30} GiB shard exceed "
                          f"40% of the host's {host_total >> 30} GiB (or the {E2E_MAX_STATE_BYTES >> 30} GiB cap)"}
    elif dist and not args.no_e2e:
        # every rank uploads its shard of the initial state (natural order of
        # the first layout) from pinned host memory, runs all parts and
        # switches, and downloads its final shard; max over ranks
        run_e2e = ShardedRun(circuit, part, int(math.log2(world)), device=dev, basis_start=False)
        run_e2e.transport, run_e2e._peer = run.transport, run._peer  # one staging pair per rank
        run_e2e._scratch = getattr(run, "_scratch", None)  # one ping-pong scratch per rank, not two
        host_in = torch.zeros(1 << n_local, dtype=torch.complex128).pin_memory()
        if rank == 0:
            host_in[0] = 1.0
        host_out = torch.empty(1 << n_local, dtype=torch.complex128).pin_memory()

        def e2e_step():
            state.copy_(host_in, non_blocking=True)
            out = run_e2e.run(state)
            host_out.copy_(out, non_blocking=True)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e_ms = float(t.item())
        nl_e2e = sum(pr.num_launches for pr in run_e2e.programs if pr is not None)
        e2e = {"value": world * num_parts * (1 << n_local) / (e_ms / 1e3) / 1e9, "unit": UNIT,
               "hbm_gbs_moved": world * nl_e2e * bytes_per_pass / (e_ms / 1e3) / 1e9,
               "launches_per_step": nl_e2e, "ms_per_step": e_ms,
               "h2d_bytes_per_step": world * (1 << n_local) * 16, "d2h_bytes_per_step": world * (1 << n_local) * 16,
               "path": "public API ShardedRun.run per rank: shard uploaded from pinned host, every part and "
                       "layout switch, shard downloaded; max over ranks"}
    if not dist and not args.no_e2e:
        shard_bytes = (1 << n) * 16
        if shard_bytes > E2E_MAX_STATE_BYTES:
            e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                   "skipped": f"a {shard_bytes >> 30} GiB state needs three device buffers and two pinned host "
                              f"buffers of its size for the overlapped stream (host RAM); measured up to "
                              f"{E2E_MAX_STATE_BYTES >> 30} GiB"}
        else:
            # a caller's initial state arrives in natural order: the e2e
            # program is planned without an initial layout of its own
            run_e2e = HierarchicalRun(circuit, part, device=dev, options=args.plan_options, basis_start=False)
            if run_e2e.program.needs_scratch and run.program.needs_scratch:
                run_e2e.program.share_scratch(run.program._scratch)
            # one pinned host input and one output (16 GiB each at c3);
            # three device buffers let the streams overlap step i+1's
            # upload, step i's passes and step i-1's download
            host_in = torch.zeros(1 << n, dtype=torch.complex128).pin_memory()
            host_in[0] = 1.0
            host_out = torch.empty(1 << n, dtype=torch.complex128).pin_memory()
            bufs = [state, torch.empty_like(state), torch.empty_like(state)]

            def e2e_steps(k):
                run_e2e.run_stream([host_in] * k, [host_out] * k, buffers=bufs, stream=stream)

            e2e_steps(max(2, args.warmup))
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_steps(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
            e_ms = e0.elapsed_time(e1) / args.steps
            assert abs(float(host_out.abs().pow(2).sum()) - 1.0) < 1e-9
            nl_e2e = run_e2e.program.num_launches
            e2e = {"value": num_parts * (1 << n_local) / (e_ms / 1e3) / 1e9, "unit": UNIT,
                   "hbm_gbs_moved": nl_e2e * bytes_per_pass / (e_ms / 1e3) / 1e9,
                   "launches_per_step": nl_e2e, "ms_per_step": e_ms, "h2d_bytes_per_step": shard_bytes,
                   "d2h_bytes_per_step": shard_bytes,
                   "path": "public API HierarchicalRun.run_stream: each step uploads an initial state from pinned "
                           "host, runs every pass and downloads the final state; upload/passes/download of "
                           "consecutive steps overlap on three streams over three device buffers"}
            del bufs, run_e2e

    info = ([run.program.info(i) for i in range(num_launches)] if not dist else run.part_infos())
    # FP64 roofline: issued FP64 pipe work of the part kernels vs a measured DFMA peak
    import ctypes

    peak = ctypes.c_double()
    _native.check(_native.load().hs_fp64_peak(ctypes.byref(peak), stream.cuda_stream))
    fp64_instr = sum(i["fp64_instr_per_amp"] for i in info) * (1 << n_local)
    part_ms = sum(durs) / n_marked if durs else (seg_ms / n_marked if dist else ms_step)
    fp64 = {"bound_note": "random-circuit passes are FP64-bound, not HBM-bound (SURVEY.md 7.3)",
            "instr_per_step": fp64_instr, "achieved_tflops": 2 * fp64_instr / (part_ms / 1e3) / 1e12,
            "peak_tflops_measured": peak.value,
            "frac": (2 * fp64_instr / (part_ms / 1e3) / 1e12) / peak.value if peak.value else None,
            "part_kernel_ms_per_step": part_ms}
    comm = None
    if dist:
        sw = [sum(c) / len(c) for c in zip(*switch_list)] if switch_list and switch_list[0] else []
        sw_ms = sum(sw)
        # switches fused into the previous segment's last launch move their
        # bytes inside that launch (counted in parts time): the NVLink rate is
        # over the separate switches only
        order = sorted(run.switch_at)
        fused = [a in getattr(run, "_fused", {}) for a in order]
        sep_bytes = sum(st.bytes_remote for st, f in zip(run.stats.switches, fused) if not f)
        sep_ms = sum(t for t, f in zip(sw, fused) if not f)
        comm = dict(run.comm_summary(), transport=run.transport, transport_note=run.transport_note,
                    switch_ms_per_step=sw_ms, per_switch_ms=[round(x, 4) for x in sw], fused=fused,
                    parts_ms_per_step=seg_ms / n_marked,
                    nvlink_gbs_per_rank=(sep_bytes / world / (sep_ms / 1e3) / 1e9 if sep_ms > 0 and sep_bytes else None),
                    nvlink_note="bytes each rank sends over the separate (unfused) switches (closed-form CommStats / "
                                "ranks) / their time; fused switches ride on the preceding pass's stores")
    if dist:
        for r_ in (run, locals().get("run_e2e")):
            if r_ is not None:
                r_.release()
    return {
        "ms_step": ms_step, "value": value, "hbm_gbs": hbm_gbs, "moved": moved, "durations_ms": durs, "bytes_per_pass": bytes_per_pass,
        "launch_ms": [sum(c) / len(c) for c in zip(*launch_ms)] if launch_ms else [],
        "num_parts": num_parts, "clocks": clk, "e2e": e2e, "info": info, "n_local": n_local,
        "num_launches": num_launches, "restore_ms_per_step": restore_ms / n_marked if n_marked else 0.0,
        "fp64": fp64, "init_ms_per_step": init_ms, "plan_s": plan_s, "jit": jit_stats, "literal": literal,
        "comm": comm,
    }


#: largest single-GPU state the e2e leg streams (three device buffers, two
#: pinned host buffers of the state's size)
E2E_MAX_STATE_BYTES = 32 << 30


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--config", default="c3", help="BASELINE config (c1 .. c5; c3 is the largest single-GPU one)")
    ap.add_argument("--strategy", default="dfs", choices=["nat", "dfs", "dagp"])
    ap.add_argument("--limit", type=int, default=None, help="part size k (default: the config's)")
    ap.add_argument("--partition", default=None, help="run this partition JSON instead of --strategy")
    ap.add_argument("--cpu-step-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-literal", action="store_true", help="skip the one-pass-per-part comparison run")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the program's kernels one by one instead of as one CUDA graph")
    ap.add_argument("--plan-add", type=lambda x: int(x, 0), default=0,
                    help="HS_PLAN_* bits added to the engine defaults (e.g. 0x400 = HS_PLAN_MERGE)")
    ap.add_argument("--plan-options", type=lambda x: int(x, 0), default=None,
                    help="planner option bits (HS_PLAN_*) of the single-GPU program (default: the engine "
                         "default + JIT + LAYOUT, chosen by state size)")
    ap.add_argument("--no-warm-plan", action="store_true", help="skip the second-process planning probe")
    ap.add_argument("--plan-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.plan_add:
        from paper_2205_06973_b200 import _native

        _native._default_options |= args.plan_add
    if args.warmup < 3 and not args.plan_probe:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    from paper_2205_06973_b200 import configs

    args.workload, scaling = configs.bench_workload(args.config, max(world, args.gpus if args.impl == "reference"
                                                                      else world))
    if args.plan_probe:
        return plan_probe(args)
    if world > 1:
        import torch.distributed as tdist

        if args.impl == "reference":
            if rank != 0:
                return 0
        else:
            tdist.init_process_group(os.environ.get("HISVSIM_BENCH_BACKEND", "nccl"))
    if args.impl == "reference":
        world = 1
    cfg, circuit, part, t_part = build_workload(args.workload, args.strategy, args.limit, args.partition)
    n = circuit.num_qubits
    gpus = args.gpus if args.impl == "reference" else world
    p_bits = int(math.log2(gpus))
    config = {"workload": f"{args.workload}: {cfg.description}" + (f", at {n} qubits" if args.workload != cfg.name
                                                                    else ""),
              "config": args.config, "num_qubits": n, "limit": args.limit or cfg.limit,
              "strategy": f"file:{Path(args.partition).name}" if args.partition else args.strategy,
              "parts": part.num_parts, "gates": circuit.num_ops, "seed": cfg.seed, "dtype": "complex128",
              "state_bytes_per_gpu": (1 << (n - p_bits)) * 16,
              "l2_policy": ("inputs larger than L2: the state exceeds the 126 MB L2" if (1 << (n - p_bits)) * 16 > (126 << 20)
                            else "L2-resident state (16 MiB c1): no flush between steps"),
              "parallelism": f"qubit-sharded x{gpus}" if gpus > 1 else "single GPU"}

    if args.impl == "reference":
        r = cpu_arm(args, cfg, circuit, part, t_part, args.steps, args.warmup)
        np_c1 = numpy_port_c1_seconds()
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator)",
                "config": config, "impl": "reference",
                "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "port",
                                 "sample": r["sample"], "numpy_port_c1_seconds": np_c1, "gbs": r["gbs"]},
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "value_definition": "amplitude updates (2 x 16 B each) / time on the sampled fixings",
                "hbm_gbs_moved": r["gbs"],
                "projected_time_to_solution_s": r["projected_time_to_solution_s"],
                "host_seconds": {"partition": round(t_part, 4)},
                "note": "host CPU, rank 0 only: the C restatement of the reference's per-part gather/gates/scatter "
                        "(oracle/sv_oracle.c; the reference is pure Python/numpy and compiles to nothing) on every "
                        "host thread over a bounded sample of each part's fixings; numpy_port_c1_seconds = the "
                        "reference's numpy algorithm (oracle/hisim_oracle.py) on all of c1, one core"}
        print(json.dumps(line), flush=True)
        return 0

    # cold planning: a fresh on-disk cubin cache for this process
    if "HISVSIM_CACHE_DIR" not in os.environ:
        import tempfile

        os.environ["HISVSIM_CACHE_DIR"] = tempfile.mkdtemp(prefix="hisvsim_bench_cache_")
    g = gpu_arm(args, circuit, part, rank, world)
    if rank != 0:
        return 0
    warm = _warm_plan_seconds(args) if world == 1 and not args.no_warm_plan else None
    peak, peak_kind = _peaks()
    durs = g["durations_ms"]
    # average duration of a launch over the timed region (every launch is one
    # pass over the shard: tile passes and gate-free layout launches alike)
    avg_ms = g["ms_step"] / max(1, g["num_launches"])
    achieved = g["bytes_per_pass"] / (avg_ms / 1e3) / 1e9
    traffic = _traffic_from_profiles(args.workload, args.strategy)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "kernel": "compiled part kernel hs_jit_part (one launch = one pass over the shard)",
                "algorithmic_bytes_per_launch": g["bytes_per_pass"],
                "avg_launch_ms": avg_ms, "launches_per_step": g["num_launches"],
                "gate_launches_per_step": sum(1 for i in g["info"] if i["user_part"] >= 0),
                "part_passes_per_step": g["num_parts"],
                "per_part_gbs": [g["bytes_per_pass"] / (d / 1e3) / 1e9 if d > 0 else None
                                 for d in durs[: g["num_parts"]]],
                "per_launch_ms": [round(x, 4) for x in g["launch_ms"]],
                "per_launch_gbs": [round(g["bytes_per_pass"] / (x / 1e3) / 1e9, 1) for x in g["launch_ms"] if x > 0]}
    infos = g["info"]
    flops = sum(i["fp_ops_per_amp"] for i in infos) * (1 << g["n_local"])
    # binding roofline per launch: max(bytes / HBM peak, FP64
    # instructions / measured DFMA rate); its sum over the circuit vs the
    # measured step
    fp_rate = g["fp64"]["peak_tflops_measured"] * 1e12 / 2  # instructions/s (FMA = 2 flops)
    bind_ms = 0.0
    for i in (infos if world == 1 else []):
        ins = i["fp64_instr_per_amp"] * (1 << g["n_local"])
        bind_ms += max(g["bytes_per_pass"] / (peak * 1e9), ins / fp_rate if fp_rate else 0.0) * 1e3
    if world == 1:
        roofline["binding"] = {"what": "sum over launches of max(HBM bytes / peak, FP64 instructions / measured DFMA rate)",
                               "bound_ms_per_step": bind_ms, "measured_ms_per_step": g["ms_step"],
                               "frac": bind_ms / g["ms_step"],
                               "fp64_instr_per_amp_per_launch": [round(i["fp64_instr_per_amp"], 1) for i in infos],
                               "hbm_ms_per_launch_at_peak": g["bytes_per_pass"] / (peak * 1e9) * 1e3,
                               "note": "a launch whose FP64 work takes longer than its HBM traffic at the measured rates "
                                       "is bound by the FP64 pipe (DFMA; B200 has no FP64 tensor-core path worth using, "
                                       "DESIGN 3.5): its HBM fraction is below 1 by construction"}
    line = {"metric": METRIC, "value": g["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": g["ms_step"], "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, no dataset)",
            "config": config,
            "launch": ("per-kernel" if (args.no_graph or world > 1) else "one CUDA graph per step (PartProgram.run_graph)"),
            "plan_add": hex(args.plan_add),
            "value_definition": "reference work rate: parts x 2^n amplitude updates per circuit (every part of the "
                                "reference partition updates every amplitude once; all ranks) / device time-to-solution "
                                "of the circuit",
            "hbm_gbs_moved": g["hbm_gbs"],
            "hbm_gbs_moved_definition": "HBM bytes the launches move (launches x 2 x 2^l x 16 B, all ranks) / step time; "
                                        "never above the HBM peak",
            "roofline": roofline, "clocks": g["clocks"],
            "gpu_launches": args.steps * g["num_launches"],
            "layout_restore_ms_per_step": g["restore_ms_per_step"],
            "init_ms_per_step": g["init_ms_per_step"],
            "e2e": g["e2e"],
            "time_to_solution_ms": g["ms_step"],
            "host_seconds": {"partition": round(t_part, 4), "plan_cold": round(g["plan_s"], 4),
                             "plan_cold_jit": g["jit"], "plan_second_process": warm,
                             "note": "plan = planner + NVRTC of every pass; cold = empty on-disk cubin cache; "
                                     "second process = the same plan in a new process that finds the cubins"},
            "one_pass_per_part": g["literal"],
            "fp64_flops_per_step_paper_count": flops,
            "fp64": g["fp64"],
            "phases_per_launch": [i["phases"] for i in infos],
            "launches_per_step": g["num_launches"],
            "comm": g["comm"]}
    if not args.no_cpu_baseline and world == 1:
        r = cpu_arm(args, cfg, circuit, part, t_part, 2, 1)
        line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "port",
                                "sample": r["sample"], "numpy_port_c1_seconds": numpy_port_c1_seconds(),
                                "gbs": r["gbs"]}
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
