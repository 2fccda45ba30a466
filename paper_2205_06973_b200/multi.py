"""One process per GPU: qubit-sharded execution with NCCL layout remaps.

The multi-GPU form of ``hisim.dist.simulate_distributed``
(/root/reference/pkg/src/hisim/dist.py:485-529), where the reference's
emulated rank axis becomes real ranks of a ``torch.distributed`` group:

* rank r owns the 2^l amplitudes whose rank qubits spell r; every part runs
  on the local shard with the same op list (one part-kernel pass);
* a layout switch old -> new moves the c qubits A = new.process & old.local
  out of the shard and brings B = old.process & new.local in. Each rank
  (1) permutes its shard so the A bits are the top c offset bits
      (hs_bit_permute) - segment k (A values = k) is then contiguous and
      bound for exactly one peer;
  (2) exchanges the 2^c segments with batched P2P send/recv (one NCCL group
      call; a segment bound for itself is a local copy);
  (3) permutes the received buffer - low bits = old.local minus A, high bits =
      B in ascending order - into the new offset order (hs_bit_permute).
  Traffic per rank = (1 - 2^-c) of its shard, the closed-form CommStats
  of ``dist.switch_stats``.

The exchange schedule is host logic shared by every back end; the local
permutations and part passes are device kernels (``DeviceOps``). Tests on a
CPU-only machine drive the same schedule over gloo with host stand-ins for
the two local operations.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import _native
from .dist import CommStats, DistributedRun, RankLayout, _part_exes, plan_layouts, storage_order
from .hier import PartProgram


@dataclass
class Segment:
    """One contiguous slice of the packed shard and where it goes."""

    index: int     # value of the A qubits (segment position in the packed shard)
    peer: int      # destination rank


def switch_schedule(old: RankLayout, new: RankLayout, rank: int):
    """For ``rank``: the packed storage order, the outgoing segments, the
    incoming segments (source rank -> slot in the receive buffer) and the
    receive-buffer storage order (low: kept locals, high: B qubits)."""
    A = [q for q in old.local if q in new.process]
    B = [q for q in old.process if q in new.local]
    kept = [q for q in old.local if q not in A]
    c = len(A)
    packed_order = tuple(kept + A)
    recv_order = tuple(kept + B)
    out = []
    for k in range(1 << c):
        dst = 0
        for bit, q in enumerate(new.process):
            if q in A:
                v = (k >> A.index(q)) & 1
            else:
                v = (rank >> old.rank_bit_of(q)) & 1
            dst |= v << bit
        out.append(Segment(k, dst))
    incoming = {}
    # sources: ranks that agree with me on the qubits staying rank bits and
    # carry any values of B; the slot is the B values of the source
    for src in range(old.num_ranks):
        for seg in switch_out_peers(old, new, src, A):
            if seg[1] == rank:
                slot = 0
                for j, q in enumerate(B):
                    slot |= ((src >> old.rank_bit_of(q)) & 1) << j
                incoming[src] = slot
    return packed_order, out, incoming, recv_order, c


def switch_out_peers(old: RankLayout, new: RankLayout, src: int, A):
    for k in range(1 << len(A)):
        dst = 0
        for bit, q in enumerate(new.process):
            v = (k >> A.index(q)) & 1 if q in A else (src >> old.rank_bit_of(q)) & 1
            dst |= v << bit
        yield k, dst


class DeviceOps:
    """Local operations on a rank's CUDA shard (libhisvsim kernels)."""

    def permute(self, src, old_order, new_order):
        from .dist import permute_storage

        return permute_storage(src, old_order, new_order)

    def empty_like(self, t):
        import torch

        return torch.empty_like(t)


class ShardedRun:
    """Plan once (layouts, switch schedules, one device program over all
    parts in rank-local coordinates), run many times."""

    def __init__(self, circuit, partition, num_rank_bits: int, group=None, device=None, ops=None,
                 dtype="complex128", program=True):
        import torch.distributed as dist

        self.circuit = circuit
        self.partition = partition
        self.p = num_rank_bits
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if self.world != 1 << num_rank_bits:
            raise ValueError(f"{self.world} ranks cannot hold {num_rank_bits} rank bits")
        self.n = circuit.num_qubits
        self.n_local = self.n - num_rank_bits
        self.first, self.layouts, switches = plan_layouts(circuit, partition, num_rank_bits)
        self.switch_at = {i: (old, new, st) for i, old, new, st in switches}
        self.exes, self.bounds = [], []
        for i, lay in enumerate(self.layouts):
            e = _part_exes(circuit, partition, i, lay)
            self.bounds.append((len(self.exes), len(e)))
            self.exes += e
        self.program = (PartProgram(self.n_local, self.exes, dtype=dtype, device=device,
                                    options=_native.default_options() & ~_native.HS_PLAN_LAYOUT)
                        if program and self.exes else None)
        self.ops = ops or DeviceOps()
        self.stats = CommStats(self.n, num_rank_bits, len(self.layouts),
                               [st for _, _, st in self.switch_at.values()])

    def part_infos(self):
        return [self.program.info(i) for i in range(len(self.exes))]

    def comm_summary(self) -> dict:
        return {"switches": self.stats.num_switches, "bytes_remote_total": self.stats.total_bytes,
                "remote_fraction_of_state": self.stats.total_bytes / float((1 << self.n) * 16)}

    def _exchange(self, packed, recv, out_segs, incoming, c):
        """Batched P2P: my segment k -> peer; slot j of recv <- source."""
        import torch.distributed as dist

        seg = packed.numel() >> c
        reqs = []
        for s in out_segs:
            chunk = packed[s.index * seg:(s.index + 1) * seg]
            if s.peer == self.rank:
                slot = incoming[self.rank]
                recv[slot * seg:(slot + 1) * seg].copy_(chunk)
            else:
                reqs.append(dist.P2POp(dist.isend, _wire(chunk), s.peer, self.group))
        for src, slot in incoming.items():
            if src != self.rank:
                reqs.append(dist.P2POp(dist.irecv, _wire(recv[slot * seg:(slot + 1) * seg]), src, self.group))
        if reqs:
            for w in dist.batch_isend_irecv(reqs):
                w.wait()

    def switch(self, shard, old: RankLayout, new: RankLayout):
        """Layout switch of this rank's shard; returns the new shard."""
        packed_order, out_segs, incoming, recv_order, c = switch_schedule(old, new, self.rank)
        old_order = tuple(old.local)
        packed = self.ops.permute(shard, old_order, packed_order)
        recv = shard  # the old shard is dead once packed: receive into it
        self._exchange(packed, recv, out_segs, incoming, c)
        return self.ops.permute(recv, recv_order, tuple(new.local))

    def run(self, shard, events=None, run_part=None):
        """All parts in order on this rank's shard (switches included);
        returns the final shard (a new tensor after any switch)."""
        import torch

        for i in range(len(self.layouts)):
            if i in self.switch_at:
                old, new, _ = self.switch_at[i]
                shard = self.switch(shard, old, new)
            start, count = self.bounds[i]
            if count:
                if run_part is not None:
                    for j in range(start, start + count):
                        run_part(shard, self.exes[j])
                else:
                    self.program.run(shard, start, count)
            if events is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                events.append(ev)
        return shard


def _wire(t):
    """complex tensors travel as their real view (NCCL has no complex type)."""
    import torch

    return torch.view_as_real(t) if t.is_complex() else t


@dataclass
class ShardedState:
    """This rank's shard of a distributed state plus the layout it is in."""

    num_qubits: int
    data: object
    layout: RankLayout
    rank: int


def simulate_distributed_group(circuit, partition, num_rank_bits, *, group=None, initial=None, dtype="complex128",
                               device=None) -> DistributedRun:
    """``simulate_distributed`` over a process group: every rank returns its
    own shard (``DistributedRun.state`` is a ``ShardedState``)."""
    import torch

    from .statevec import allocate, init_basis

    run = ShardedRun(circuit, partition, num_rank_bits, group=group, device=device, dtype=dtype)
    shard = allocate(run.n_local, dtype, device)
    if initial is None:
        if run.rank == 0:
            init_basis(shard, 0)
        else:
            shard.zero_()
    else:
        raise NotImplementedError("initial= with a process group: load each rank's shard instead")
    shard = run.run(shard)
    torch.cuda.synchronize()
    return DistributedRun(ShardedState(run.n, shard, run.layouts[-1], run.rank), run.stats, run.layouts)


def shard_positions(layout: RankLayout, rank: int):
    """Global index of every offset of ``rank``'s shard (host, small n)."""
    import numpy as np

    off = np.arange(1 << layout.num_local_qubits, dtype=np.int64)
    g = np.zeros_like(off)
    for j, q in enumerate(layout.local):
        g |= ((off >> j) & 1) << q
    for k, q in enumerate(layout.process):
        g |= np.int64(((rank >> k) & 1) << q)
    return g


__all__ = ["ShardedRun", "ShardedState", "DeviceOps", "switch_schedule", "simulate_distributed_group",
           "shard_positions", "storage_order", "math"]
