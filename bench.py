"""Benchmark: circuit time-to-solution and effective HBM GB/s per part-pass.

One step = one full simulation of the BASELINE config circuit (every part
of its partition, one kernel pass each) on a state already resident in HBM.
``value`` = algorithmic part-pass bytes of all ranks / step time, where a
part-pass moves 2 x 2^l x 16 B (read + write of a rank's shard, SURVEY.md
§8(d)); ``ms_per_step`` is the circuit time-to-solution (partitioning, done
once on the host, is reported separately). ``e2e`` is the same metric
through the public API with the initial state in pinned host memory and the
final state read back every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--strategy dfs]
    python bench.py --impl reference ...   # the CPU port of the reference path

Under torchrun (N > 1) the state is sharded over the N ranks (n + log2 N
qubits, weak scaling) and layout switches run over NCCL.
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
UNIT = "GB/s"


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
        if d.get("workload") == f"{config}/{strategy}" and d.get("dram_bytes_per_launch"):
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


def build_workload(config: str, strategy: str, extra_bits: int = 0, limit: int | None = None):
    from paper_2205_06973_b200 import build_dag, configs, partition_dagp, partition_dfs, partition_nat

    cfg = configs.CONFIGS[config.split("@")[0]]
    name = config
    if extra_bits:
        name = f"{config.split('@')[0]}@{cfg.num_qubits + extra_bits}"
    circuit = configs.build(name)
    t0 = time.perf_counter()
    fn = {"nat": partition_nat, "dfs": partition_dfs, "dagp": partition_dagp}[strategy]
    part = fn(build_dag(circuit), limit or cfg.limit)
    t_part = time.perf_counter() - t0
    return cfg, circuit, part, t_part


# --------------------------------------------------------------------------- CPU reference arm

def cpu_arm(args, cfg, circuit, part, t_part, steps, warmup, quiet=False):
    """The reference path's CPU restatement (oracle/sv_oracle.c, all host
    threads) on a bounded sample of fixings of every part."""
    import numpy as np

    from oracle import c_oracle

    c_oracle.lib()
    threads = c_oracle.threads()
    n = circuit.num_qubits
    # calibrate: fixings per part so that one step takes ~target seconds
    target = args.cpu_step_seconds
    psi = np.empty(1 << n, dtype=np.complex128)
    psi.fill(0)  # fault the pages in before timing anything
    psi[0] = 1.0
    slots = [c_oracle.part_slots(circuit, p.gate_indices, p.qubits) for p in part.parts]
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
    value = nbytes / dt / 1e9
    sample_amps = sum(k << len(pos) for pos, _, _, k in plan)
    sample = (f"{config_label(args)}: each step runs every one of the {len(plan)} parts over "
              f"{sample_amps / (1 << n) / len(plan):.4%} of its fixings ({sample_amps} amplitude updates "
              f"per step, fixings 0..k-1 of each part) with {threads} threads; GB/s = 2 x 16 B x "
              f"amplitudes / time, the same algorithmic count as the GPU arm")
    full_s = (len(plan) * (1 << n) * 32) / (value * 1e9)
    return {
        "value": value, "threads": threads, "sample": sample, "ms_per_step": dt / steps * 1e3,
        "projected_time_to_solution_s": full_s,
    }


def config_label(args):
    return f"{args.config}/{args.strategy}"


# --------------------------------------------------------------------------- GPU arm

def gpu_arm(args, cfg, circuit, part, t_part, rank, world):
    import numpy as np
    import torch

    from paper_2205_06973_b200.hier import HierarchicalRun, execute_hierarchical
    from paper_2205_06973_b200.statevec import allocate, init_basis

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    n = circuit.num_qubits
    dist = world > 1
    if dist:
        from paper_2205_06973_b200.multi import ShardedRun

        run = ShardedRun(circuit, part, int(math.log2(world)), device=dev)
        n_local = run.n_local
    else:
        # the timed runs start from |0..0>, prepared in the program's layout
        run = HierarchicalRun(circuit, part, device=dev, options=args.plan_options, basis_start=True)
        n_local = n
    num_parts = part.num_parts
    num_launches = (run.program.num_launches if not dist
                    else sum(pr.num_launches for pr in run.programs if pr is not None))
    bytes_per_pass = 2 * (1 << n_local) * 16
    launch_owner = [run.program.info(j)["user_part"] for j in range(num_launches)] if not dist else []
    state = allocate(n_local, "complex128", dev)
    stream = torch.cuda.current_stream(dev)

    # the whole program as one CUDA graph launch (PartProgram.run_graph,
    # captured in the warm-up) unless --no-graph: launch overhead matters for
    # L2-resident states (c1: 7 launches of ~16 us)
    def launch(buf):
        if args.no_graph:
            run.program.run(buf)
        else:
            run.program.run_graph(buf, stream=stream)

    def one_step(timed_events=None):
        if not dist:
            run.program.init_basis(state, 0)
        elif rank == 0:
            init_basis(state, 0)
        else:
            state.zero_()
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
    # all parts (and switches) run between two events on the launch stream
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for e_init, e0, e1 in step_ev:
        e_init.record(stream)
        if not dist:
            run.program.init_basis(state, 0)
        elif rank == 0:
            init_basis(state, 0)
        else:
            state.zero_()
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
    # per-launch durations of the part kernel (events between launches);
    # distributed: per segment ("parts") and per layout switch ("switch")
    durs, restore_ms, switch_ms, seg_ms = [], 0.0, 0.0, 0.0
    launch_ms = []  # per launch, per marked step
    for ev in marks:
        if dist:
            for i in range(1, len(ev)):
                kind, e = ev[i]
                prev = ev[i - 1][1] if isinstance(ev[i - 1], tuple) else ev[i - 1]
                if kind == "switch":
                    switch_ms += prev.elapsed_time(e)
                else:
                    seg_ms += prev.elapsed_time(e)
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
    value = world * num_parts * bytes_per_pass / (ms_step / 1e3) / 1e9

    # e2e through the public API: host initial state in, host state out
    e2e = None
    if dist and not args.no_e2e:
        # every rank uploads its shard of the initial state (natural order of
        # the first layout) from pinned host memory, runs all parts and
        # switches, and downloads its final shard; max over ranks
        run_e2e = ShardedRun(circuit, part, int(math.log2(world)), device=dev, basis_start=False)
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
        e2e = {"value": world * num_parts * bytes_per_pass / (e_ms / 1e3) / 1e9, "unit": UNIT,
               "launches_per_step": sum(pr.num_launches for pr in run_e2e.programs if pr is not None),
               "ms_per_step": e_ms, "h2d_bytes_per_step": world * (1 << n_local) * 16,
               "d2h_bytes_per_step": world * (1 << n_local) * 16,
               "path": "public API ShardedRun.run per rank: shard uploaded from pinned host, every part and "
                       "layout switch, shard downloaded; max over ranks"}
    if not dist and not args.no_e2e:
        # a caller's initial state arrives in natural order: the e2e program
        # is planned without an initial layout of its own
        run_e2e = HierarchicalRun(circuit, part, device=dev, options=args.plan_options, basis_start=False)
        # pinned host inputs / outputs alternate; three device buffers let
        # the streams overlap step i+1's upload, step i's parts and step
        # i-1's download
        host_in = [torch.zeros(1 << n, dtype=torch.complex128).pin_memory() for _ in range(2)]
        for h in host_in:
            h[0] = 1.0
        host_out = [torch.empty(1 << n, dtype=torch.complex128).pin_memory() for _ in range(2)]
        bufs = [state, torch.empty_like(state), torch.empty_like(state)]

        def e2e_steps(k):
            run_e2e.run_stream([host_in[i % 2] for i in range(k)], [host_out[i % 2] for i in range(k)],
                               buffers=bufs, stream=stream)

        e2e_steps(max(2, args.warmup))
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_steps(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.steps
        for h in host_out:
            assert abs(float(h.abs().pow(2).sum()) - 1.0) < 1e-9
        e2e = {"value": num_parts * bytes_per_pass / (e_ms / 1e3) / 1e9, "unit": UNIT,
               "launches_per_step": run_e2e.program.num_launches,
               "ms_per_step": e_ms, "h2d_bytes_per_step": (1 << n) * 16, "d2h_bytes_per_step": (1 << n) * 16,
               "path": "public API HierarchicalRun.run_stream: each step uploads an initial state from pinned host, "
                       "runs every part and downloads the final state; upload/parts/download of consecutive "
                       "steps overlap on three streams over three device buffers"}

    info = ([run.program.info(i) for i in range(num_launches)] if not dist else run.part_infos())
    # FP64 roofline: issued FP64 pipe work of the part kernels vs a measured DFMA peak
    import ctypes

    from paper_2205_06973_b200 import _native

    peak = ctypes.c_double()
    _native.check(_native.load().hs_fp64_peak(ctypes.byref(peak), stream.cuda_stream))
    fp64_instr = sum(i["fp64_instr_per_amp"] for i in info) * (1 << n_local)
    part_ms = sum(durs) / n_marked if durs else (seg_ms / n_marked if dist else ms_step)
    fp64 = {"bound_note": "random-circuit parts are FP64-bound, not HBM-bound (SURVEY.md 7.3)",
            "instr_per_step": fp64_instr, "achieved_tflops": 2 * fp64_instr / (part_ms / 1e3) / 1e12,
            "peak_tflops_measured": peak.value,
            "frac": (2 * fp64_instr / (part_ms / 1e3) / 1e12) / peak.value if peak.value else None,
            "part_kernel_ms_per_step": part_ms}
    return {
        "ms_step": ms_step, "value": value, "durations_ms": durs, "bytes_per_pass": bytes_per_pass,
        "launch_ms": [sum(c) / len(c) for c in zip(*launch_ms)] if launch_ms else [],
        "num_parts": num_parts, "clocks": clk, "e2e": e2e, "info": info, "n_local": n_local,
        "num_launches": num_launches, "restore_ms_per_step": restore_ms / n_marked, "fp64": fp64,
        "init_ms_per_step": init_ms,
        "comm": (dict(run.comm_summary(), switch_ms_per_step=switch_ms / n_marked,
                      parts_ms_per_step=seg_ms / n_marked,
                      nvlink_gbs_per_rank=(run.stats.total_bytes / world / (switch_ms / n_marked / 1e3) / 1e9
                                           if switch_ms > 0 else None))
                 if dist else None),
    }


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--strategy", default="dfs", choices=["nat", "dfs", "dagp"])
    ap.add_argument("--limit", type=int, default=None, help="part size k (default: the config's)")
    ap.add_argument("--cpu-step-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the program's kernels one by one instead of as one CUDA graph")
    ap.add_argument("--plan-add", type=lambda x: int(x, 0), default=0,
                    help="HS_PLAN_* bits added to the engine defaults (e.g. 0x400 = HS_PLAN_MERGE)")
    ap.add_argument("--plan-options", type=lambda x: int(x, 0), default=None,
                    help="planner option bits (HS_PLAN_*) of the single-GPU program (default: the engine "
                         "default + JIT + LAYOUT, chosen by state size)")
    args = ap.parse_args(argv)
    if args.plan_add:
        from paper_2205_06973_b200 import _native

        _native._default_options |= args.plan_add
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as tdist

        if args.impl == "reference":
            if rank != 0:
                return 0
        else:
            tdist.init_process_group("nccl")
    # weak scaling: n + log2 N qubits (the reference arm times the same
    # workload on rank 0's host cores)
    extra = int(math.log2(world)) if world > 1 else 0
    if args.impl == "reference":
        world = 1
    cfg, circuit, part, t_part = build_workload(args.config, args.strategy, extra, args.limit)
    n = circuit.num_qubits
    config = {"workload": f"{args.config}: {cfg.description}" + (f", scaled to {n} qubits" if extra else ""),
              "num_qubits": n, "limit": args.limit or cfg.limit, "strategy": args.strategy, "parts": part.num_parts,
              "gates": circuit.num_ops, "seed": cfg.seed, "dtype": "complex128",
              "state_bytes_per_gpu": (1 << (n - extra)) * 16,
              "l2_policy": "inputs larger than L2: the state (>= 1 GiB) exceeds the 126 MB L2",
              "partition_seconds_host": round(t_part, 4), "plan_add": hex(args.plan_add),
              "launch": "per-kernel" if (args.no_graph or world > 1) else "one CUDA graph per step (PartProgram.run_graph)", "parallelism": (f"qubit-sharded x{world}" if world > 1 else "single GPU") if args.impl != "reference"
              else f"host CPU threads (rank 0 of {args.gpus})"}

    if args.impl == "reference":
        r = cpu_arm(args, cfg, circuit, part, t_part, args.steps, args.warmup)
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator)",
                "config": config, "impl": "reference",
                "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "port",
                                 "sample": r["sample"]},
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "projected_time_to_solution_s": r["projected_time_to_solution_s"]}
        print(json.dumps(line), flush=True)
        return 0

    g = gpu_arm(args, cfg, circuit, part, t_part, rank, world)
    if rank != 0:
        return 0
    peak, peak_kind = _peaks()
    durs = g["durations_ms"]
    # average duration of a launch that carries gates over the timed region:
    # the timed part time less the gate-free layout launches (their share
    # from the event pass). Wide parts take several launches (sub-passes,
    # regrouped across parts), so a launch is not always a part: the per
    # part-pass figure (value's unit) is reported beside it.
    gate_launches = (sum(1 for i in g["info"] if i["user_part"] >= 0) if world == 1 else g["num_parts"])
    avg_ms = (g["ms_step"] - g["restore_ms_per_step"]) / max(1, gate_launches)
    part_pass_ms = (g["ms_step"] - g["restore_ms_per_step"]) / g["num_parts"]
    achieved = g["bytes_per_pass"] / (avg_ms / 1e3) / 1e9
    traffic = _traffic_from_profiles(args.config, args.strategy)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "kernel": "compiled part kernel (one launch = one pass over the state)",
                "algorithmic_bytes_per_launch": g["bytes_per_pass"],
                "avg_launch_ms": avg_ms, "gate_launches_per_step": gate_launches,
                "part_passes_per_step": g["num_parts"],
                "effective_gbs_per_part_pass": g["bytes_per_pass"] / (part_pass_ms / 1e3) / 1e9,
                "avg_launch_ms_event_pass": (sum(durs) / len(durs)) if durs else None,
                "per_part_gbs": [g["bytes_per_pass"] / (d / 1e3) / 1e9 if d > 0 else None
                                 for d in durs[: g["num_parts"]]],
                "per_launch_ms": [round(x, 4) for x in g["launch_ms"]],
                "per_launch_gbs": [round(g["bytes_per_pass"] / (x / 1e3) / 1e9, 1) for x in g["launch_ms"] if x > 0]}
    infos = g["info"]
    flops = sum(i["fp_ops_per_amp"] for i in infos) * (1 << g["n_local"])
    # binding roofline per part: max(bytes / HBM peak, FP64
    # instructions / measured DFMA rate); its sum over the circuit vs the
    # measured part time
    fp_rate = g["fp64"]["peak_tflops_measured"] * 1e12 / 2  # instructions/s (FMA = 2 flops)
    bind_ms = 0.0
    for i in (infos if world == 1 else []):  # every launch is one pass over the state
        ins = i["fp64_instr_per_amp"] * (1 << g["n_local"])
        bind_ms += max(g["bytes_per_pass"] / (peak * 1e9), ins / fp_rate if fp_rate else 0.0) * 1e3
    if world == 1:
        roofline["binding"] = {"what": "sum over launches of max(HBM bytes / peak, FP64 instructions / measured DFMA rate)",
                             "bound_ms_per_step": bind_ms, "measured_ms_per_step": g["ms_step"],
                             "frac": bind_ms / g["ms_step"]}
    line = {"metric": METRIC, "value": g["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": g["ms_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, no dataset)",
            "config": config, "roofline": roofline, "clocks": g["clocks"],
            "gpu_launches": args.steps * g["num_launches"] + (args.steps * g["e2e"]["launches_per_step"] if g["e2e"] else 0),
            "layout_restore_ms_per_step": g["restore_ms_per_step"],
            "init_ms_per_step": g["init_ms_per_step"],
            "e2e": g["e2e"],
            "time_to_solution_ms": g["ms_step"],
            "fp64_flops_per_step_paper_count": flops,
            "fp64": g["fp64"],
            "phases_per_launch": [i["phases"] for i in infos],
            "launches_per_step": g["num_launches"],
            "comm": g["comm"]}
    if not args.no_cpu_baseline and world == 1:
        r = cpu_arm(args, cfg, circuit, part, t_part, 2, 1)
        line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "port",
                                "sample": r["sample"]}
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
