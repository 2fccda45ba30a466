"""The multi-process (one rank per GPU) remap path over gloo on CPU.

Two and four ranks run the real exchange schedule of
``paper_2205_06973_b200.multi.ShardedRun`` (batched P2P send/recv through
torch.distributed); the two rank-local operations (bit permutation and the
part pass) use host stand-ins here, the CUDA kernels on a GPU box. The
gathered shards must equal the reference's distributed result.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _compose(k, m, seg_pos, nbits):
    """index with segment bits k at seg_pos (ascending) and inner offset m elsewhere"""
    idx = np.asarray(m, dtype=np.int64).copy()
    for b, q in enumerate(seg_pos):
        lo = idx & ((1 << q) - 1)
        idx = ((idx ^ lo) << 1) | lo | (((k >> b) & 1) << q)
    return idx


class HostOps:
    """numpy stand-ins for the rank-local device kernels"""

    def empty(self, count, like):
        return torch.empty(count, dtype=like.dtype)

    def pack_range(self, shard, staging, nbits, seg_pos, begin, count):
        m = np.arange(begin, begin + count, dtype=np.int64)
        for k in range(1 << len(seg_pos)):
            staging[k * count:(k + 1) * count] = shard[torch.from_numpy(_compose(k, m, seg_pos, nbits))]

    def unpack_range(self, staging, shard, nbits, seg_pos, begin, count):
        m = np.arange(begin, begin + count, dtype=np.int64)
        for k in range(1 << len(seg_pos)):
            shard[torch.from_numpy(_compose(k, m, seg_pos, nbits))] = staging[k * count:(k + 1) * count]

    def to_natural(self, shard, phys):
        """logical position q sits on physical bit phys[q]: gather into natural order"""
        n = len(phys)
        i = np.arange(1 << n, dtype=np.int64)
        src = np.zeros_like(i)
        for q, b in enumerate(phys):
            src |= ((i >> q) & 1) << b
        return shard[torch.from_numpy(src)].clone()

    def permute(self, src, old_order, new_order):
        n = len(old_order)
        where = {q: b for b, q in enumerate(new_order)}
        i = np.arange(1 << n, dtype=np.int64)
        o = np.zeros_like(i)
        for b, q in enumerate(old_order):
            o |= ((i >> b) & 1) << where[q]
        out = np.empty(1 << n, dtype=np.complex128)
        out[o] = src.numpy()
        return torch.from_numpy(out)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, qasm, parts, p, out, policy="reference"):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import partition_of
        from oracle import hisim_oracle as orc
        from paper_2205_06973_b200.multi import ShardedRun, shard_positions
        from paper_2205_06973_b200.qasm import parse_qasm

        c = parse_qasm(qasm)
        # a tiny chunk so each switch takes several pack/exchange/unpack rounds
        run = ShardedRun(c, partition_of(parts), p, ops=HostOps(), program=False, chunk_bytes=64, policy=policy)
        shard = torch.zeros(1 << run.n_local, dtype=torch.complex128)
        if rank == 0:
            shard[0] = 1.0

        def run_part(t, exe):
            a = t.numpy()
            orc.run_part(a, exe.slot_map.qubits, exe.ops, exe.op_slots)

        shard = run.run(shard, run_part=run_part)
        pos = shard_positions(run.layouts[-1], rank)
        out[rank] = (pos, shard.numpy().copy(), run.stats.total_bytes)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,policy", [(2, "reference"), (4, "reference"), (4, "lookahead")])
def test_sharded_run_over_gloo_matches_reference(golden, world, policy):
    p = world.bit_length() - 1
    docs, states = golden.json("corpus"), golden.npz("corpus")
    picked = [(i, d) for i, doc in enumerate(docs) for d in doc["dist"] if d["p"] == p and d["switches"]][:3]
    assert picked
    ctx = mp.get_context("spawn")
    for i, d in picked:
        mgr = ctx.Manager()
        out = mgr.dict()
        port = _port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, docs[i]["qasm"], d["parts"], p, out, policy))
                 for r in range(world)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(120)
            assert pr.exitcode == 0
        n = int(np.log2(states[f"c{i}"].size))
        full = np.zeros(1 << n, dtype=np.complex128)
        for r in range(world):
            pos, amp, total = out[r]
            full[pos] = amp
        assert np.max(np.abs(full - states[f"c{i}"])) < 1e-12
        ref_bytes = sum(s["bytes_remote"] for s in d["switches"])
        if policy == "reference":  # the reference's layouts, so its CommStats exactly
            assert out[0][2] == ref_bytes
        else:  # the lookahead schedule never moves more
            assert out[0][2] <= ref_bytes


def _emulate_group_switch(shards, nbits, seg_pos, c, seg_dst, src_slot, chunk):
    """numpy model of hs_group_switch's contract (include/hisvsim.h): per
    chunk of inner offsets every shard packs its segments into staging, then
    pulls slot j from the staging segment of the shard whose data lands in
    slot j and whose segment goes here."""
    R, S = len(shards), 1 << c
    inner = 1 << (nbits - c)
    src_of = {}
    for s in range(R):
        for k in range(S):
            src_of[(seg_dst[s * S + k], src_slot[s])] = (s, k)
    for begin in range(0, inner, chunk):
        m = np.arange(begin, min(inner, begin + chunk), dtype=np.int64)
        staging = [[sh[_compose(k, m, seg_pos, nbits)].copy() for k in range(S)] for sh in shards]
        for r in range(R):
            for j in range(S):
                s, k = src_of[(r, j)]
                shards[r][_compose(j, m, seg_pos, nbits)] = staging[s][k]
    return shards


def test_group_switch_arguments_reproduce_the_reference_runs(golden):
    """multi.group_switch_args + the hs_group_switch contract (emulated in
    numpy, small chunks) with numpy part passes reproduce the reference's
    distributed states on the corpus (both remap policies)."""
    from conftest import partition_of
    from oracle import hisim_oracle as orc
    from paper_2205_06973_b200.multi import ShardedRun, group_switch_args, shard_positions
    from paper_2205_06973_b200.qasm import parse_qasm

    docs, states = golden.json("corpus"), golden.npz("corpus")
    checked = 0
    for i, doc in enumerate(docs[:40]):
        c = parse_qasm(doc["qasm"])
        for d in doc["dist"]:
            if not d["switches"]:
                continue
            for policy in ("reference", "lookahead"):
                run = ShardedRun(c, partition_of(d["parts"]), d["p"], loopback=True, program=False, policy=policy)
                R, l = 1 << d["p"], run.n_local
                shards = [np.zeros(1 << l, dtype=np.complex128) for _ in range(R)]
                shards[0][0] = 1.0
                for si, (a, b) in enumerate(run.segments):
                    if a in run.switch_at:
                        pa, cc, dst, slot = group_switch_args(run, si)
                        _emulate_group_switch(shards, l, pa, cc, dst, slot, chunk=3)
                        # the host passes address the new layout in natural order:
                        # offset bit j of it sits on physical bit arrival[j]
                        old, new, _ = run.switch_at[a]
                        arrival = run.arrival_layout(old, new)
                        idx = np.arange(1 << l, dtype=np.int64)
                        src = np.zeros_like(idx)
                        for j, ph in enumerate(arrival):
                            src |= ((idx >> j) & 1) << ph
                        shards = [sh[src] for sh in shards]
                    for j in range(run.bounds[a][0], run.bounds[b - 1][0] + run.bounds[b - 1][1]) if b > a else ():
                        e = run.exes[j]
                        for sh in shards:
                            orc.run_part(sh, e.slot_map.qubits, e.ops, e.op_slots)
                full = np.zeros(1 << c.num_qubits, dtype=np.complex128)
                for r in range(R):
                    full[shard_positions(run.layouts[-1], r)] = shards[r]
                assert np.max(np.abs(full - states[f"c{i}"])) < 1e-12, (i, d["p"], policy)
                checked += 1
    assert checked >= 10
