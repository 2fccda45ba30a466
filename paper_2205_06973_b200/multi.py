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


def switch_schedule(old: RankLayout, new: RankLayout, rank: int, A=None):
    """For ``rank``: the packed storage order, the outgoing segments, the
    incoming segments (source rank -> slot in the receive buffer) and the
    receive-buffer storage order (low: kept locals, high: B qubits).
    ``A``: order of the outgoing qubits = the bits of a segment index
    (default ascending; the in-place switch orders them by physical bit)."""
    if A is None:
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

    def empty(self, count, like):
        import torch

        return torch.empty(count, dtype=like.dtype, device=like.device)

    def _range(self, fn, src, dst, num_bits, seg_pos, begin, count):
        import ctypes

        import torch

        from .statevec import native_dtype

        lib = _native.load()
        sp = (ctypes.c_int32 * max(1, len(seg_pos)))(*seg_pos)
        t = src if src.is_cuda else dst
        stream = torch.cuda.current_stream(t.device).cuda_stream
        _native.check(getattr(lib, fn)(src.data_ptr(), dst.data_ptr(), num_bits, native_dtype(t), sp, len(seg_pos),
                                       begin, count, stream))

    def pack_range(self, shard, staging, num_bits, seg_pos, begin, count):
        """staging[k * count + m] = shard[segment k, inner offset begin + m]"""
        self._range("hs_pack_segments_range", shard, staging, num_bits, seg_pos, begin, count)

    def unpack_range(self, staging, shard, num_bits, seg_pos, begin, count):
        self._range("hs_unpack_segments_range", staging, shard, num_bits, seg_pos, begin, count)


#: staging for one chunk of an in-place switch, all segments together
SWITCH_CHUNK_BYTES = 256 << 20


#: staging per buffer of the peer-memory switch (two per rank; fewer chunks
#: means fewer rank barriers)
P2P_STAGING_BYTES = 4 << 30


class PeerStaging:
    """Two staging buffers per rank (``hs_device_alloc``: whole allocations,
    so an IPC mapping's base is the buffer) exported with CUDA IPC and mapped
    by every peer (``hs_ipc_open_handle``). Setup is collective: if any rank
    fails to map any peer, every rank raises."""

    def __init__(self, nbytes: int, group=None, device=None):
        import ctypes

        import torch
        import torch.distributed as dist

        self.bytes = int(nbytes)
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._lib = lib = _native.load()
        self.local, self._opened = [], []
        self._remote = {}
        err = None
        if device is not None:
            torch.cuda.set_device(torch.device(device))
        handles = []
        try:
            # kernels here read the peers' staging and write their shards
            devs = [None] * self.world
            dist.all_gather_object(devs, torch.cuda.current_device(), group=group)
            for d in sorted(set(devs)):
                _native.check(lib.hs_enable_peer_access(int(d)))
            for _ in range(2):
                ptr = ctypes.c_void_p()
                _native.check(lib.hs_device_alloc(self.bytes, ctypes.byref(ptr)))
                self.local.append(ptr.value)
                h = ctypes.create_string_buffer(64)
                _native.check(lib.hs_ipc_get_handle(ptr, h))
                handles.append(h.raw)
        except Exception as exc:
            err = f"rank {self.rank}: {exc}"
        gathered = [None] * self.world
        dist.all_gather_object(gathered, (handles, err), group=group)
        if err is None:
            try:
                for r, (hs, e) in enumerate(gathered):
                    if r == self.rank or e is not None:
                        continue
                    for b, h in enumerate(hs):
                        ptr = ctypes.c_void_p()
                        buf = ctypes.create_string_buffer(h, 64)
                        _native.check(lib.hs_ipc_open_handle(buf, ctypes.byref(ptr)))
                        self._remote[(r, b)] = ptr.value
                        self._opened.append(ptr.value)
            except Exception as exc:
                err = f"rank {self.rank}: {exc}"
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)
        bad = [e for e in errs if e] + [e for _, e in gathered if e]
        if bad:
            self.close()
            raise RuntimeError("; ".join(sorted(set(bad))))

    def ptr(self, rank: int, b: int) -> int:
        return self.local[b] if rank == self.rank else self._remote[(rank, b)]

    def close(self) -> None:
        lib = getattr(self, "_lib", None)
        if lib is None:
            return
        for p in self._opened:
            lib.hs_ipc_close(p)
        for p in self.local:
            lib.hs_device_free(p)
        self._opened, self.local, self._remote = [], [], {}

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


class ShardedRun:
    """Plan once (layouts, switch schedules, one device program per run of
    parts between switches, in rank-local coordinates), run many times.

    Switches are in place and chunked (``switch``), so a rank needs its shard
    plus a small staging buffer: 36 qubits over 8 GPUs (128 GiB shards) fit.
    After a switch the incoming rank qubits sit on the bit positions of the
    outgoing ones; the next segment's program takes that physical layout as
    its initial layout and ends in natural order."""

    def __init__(self, circuit, partition, num_rank_bits: int, group=None, device=None, ops=None,
                 dtype="complex128", program=True, chunk_bytes: int = SWITCH_CHUNK_BYTES, basis_start: bool = True,
                 loopback: bool = False, policy: str = "lookahead", transport: str = "nccl",
                 staging_bytes: int | None = None, fuse_switches: bool = True):
        """``loopback``: all ranks live in this process on one device
        (``run_loopback``); no process group is used. ``policy``: layout
        schedule (``dist.plan_layouts``): "lookahead" (default: fewest remap
        bytes) or "reference" (the reference's layouts and CommStats)."""
        import torch.distributed as dist

        self.circuit = circuit
        self.partition = partition
        self.p = num_rank_bits
        self.group = group
        if loopback:
            self.rank, self.world = 0, 1 << num_rank_bits
        else:
            self.rank = dist.get_rank(group) if dist.is_initialized() else 0
            self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if self.world != 1 << num_rank_bits:
            raise ValueError(f"{self.world} ranks cannot hold {num_rank_bits} rank bits")
        self.n = circuit.num_qubits
        self.n_local = self.n - num_rank_bits
        self.chunk_bytes = int(chunk_bytes)
        self.policy = policy
        self.first, self.layouts, switches = plan_layouts(circuit, partition, num_rank_bits, policy)
        self.switch_at = {i: (old, new, st) for i, old, new, st in switches}
        self.exes, self.bounds = [], []
        for i, lay in enumerate(self.layouts):
            e = _part_exes(circuit, partition, i, lay)
            self.bounds.append((len(self.exes), len(e)))
            self.exes += e
        # segments: runs of parts between switches, each one device program
        starts = [0] + sorted(i for i in self.switch_at if i > 0)
        ends = starts[1:] + [len(self.layouts)]
        self.segments = list(zip(starts, ends))
        self.ops = ops or DeviceOps()
        self.programs = []
        self.seg_phys_in, self.seg_phys_out = [], []  # per segment: layout in / out (None = natural)
        if program:
            # a segment followed by a switch leaves the shard in its final
            # layout (no restore passes): the switch packs from it, and the
            # next segment starts from the layout the switch leaves
            phys = None
            for si, (a, b) in enumerate(self.segments):
                init = None
                if si > 0:
                    old, new, _ = self.switch_at[a]
                    init = self.arrival_layout(old, new, phys)
                self.seg_phys_in.append(init)
                ex = self.exes[self.bounds[a][0]:self.bounds[b - 1][0] + self.bounds[b - 1][1]] if b > a else []
                last = si + 1 == len(self.segments)
                if not ex:
                    self.programs.append(None)
                    phys = None if init is None else tuple(init)
                    if last and phys is not None:
                        raise NotImplementedError("a switch with no parts after it")
                    self.seg_phys_out.append(phys)
                    continue
                pr = PartProgram(self.n_local, ex, dtype=dtype, device=device, init_layout=init,
                                 basis_start=basis_start and si == 0, final_natural=last)
                self.programs.append(pr)
                phys = None if pr.final_layout == tuple(range(self.n_local)) else pr.final_layout
                self.seg_phys_out.append(phys)
        self.program = self.programs[0] if self.programs else None
        self.stats = CommStats(self.n, num_rank_bits, len(self.layouts),
                               [st for _, _, st in self.switch_at.values()])
        # switch transport: "nccl" (batched send/recv), "p2p" (pull from the
        # peers' staging over peer memory, CUDA IPC mappings), "auto" (p2p
        # when every rank can map every peer's staging, else nccl)
        if transport not in ("nccl", "p2p", "auto"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = "nccl"
        self.transport_note = None
        self._peer = None
        # p2p: switches fused into the last pass of the segment before them
        # (hs_program_fuse_switch), set up on the first run with a shard
        self.fuse_switches = fuse_switches
        self._fused = {}        # switch index a -> True when segment a-1's last launch performs it
        self._fused_for = None  # data_ptr of the shard the fused launches write
        self._state_maps = []   # peers' shard storages mapped through CUDA IPC (kept alive)
        if transport != "nccl" and not loopback and self.world > 1 and self.switch_at:
            amp = 16 if str(dtype) in ("complex128", "c128", "torch.complex128") else 8
            shard = amp << self.n_local
            sb = int(staging_bytes) if staging_bytes else max(SWITCH_CHUNK_BYTES, min(P2P_STAGING_BYTES, shard))
            try:
                self._peer = PeerStaging(sb, self.group, device)
                self.transport = "p2p"
            except Exception as exc:  # decided collectively inside PeerStaging
                if transport == "p2p":
                    raise
                self.transport_note = f"p2p unavailable, nccl used: {exc}"

    def _share_scratch(self, shard) -> None:
        """One ping-pong scratch buffer for all segment programs (each would
        otherwise keep its own shard-sized buffer)."""
        sc = getattr(self, "_scratch", None)
        if not any(pr is not None and pr.needs_scratch for pr in self.programs):
            return
        if sc is None or sc.numel() < shard.numel() or sc.dtype != shard.dtype or sc.device != shard.device:
            import torch

            self._scratch = sc = torch.empty(shard.numel(), dtype=shard.dtype, device=shard.device)
        for pr in self.programs:
            if pr is not None:
                pr.share_scratch(sc)

    def part_infos(self):
        """hs_part_info of every launch of every segment program (wide parts
        take several launches; gate-free layout launches report user_part -1)."""
        return [pr.info(i) for pr in self.programs if pr is not None for i in range(pr.num_launches)]

    def comm_summary(self) -> dict:
        return {"switches": self.stats.num_switches, "bytes_remote_total": self.stats.total_bytes,
                "remote_fraction_of_state": self.stats.total_bytes / float((1 << self.n) * 16),
                "fused_switches": len(self._fused)}

    @staticmethod
    def switch_plan(old: RankLayout, new: RankLayout, phys=None):
        """Physical bits of the outgoing qubits A (ascending: A is ordered by
        them) and the incoming qubits B; bit i of a segment / slot index is
        A[i] / B[i]. ``phys``: physical bit of each offset position of
        ``old`` in the shard (the previous segment's final layout; None =
        natural)."""
        at = (lambda j: j) if phys is None else (lambda j: phys[j])
        A = [q for q in old.local if q in new.process]
        A.sort(key=lambda q: at(old.local.index(q)))
        B = [q for q in old.process if q in new.local]
        pa = [at(old.local.index(q)) for q in A]
        return A, B, pa

    @classmethod
    def arrival_layout(cls, old: RankLayout, new: RankLayout, phys=None):
        """Physical offset bit of each of ``new.local``'s qubits after the
        in-place switch: kept qubits stay, B[i] lands on A[i]'s bit."""
        A, B, pa = cls.switch_plan(old, new, phys)
        where = {q: (j if phys is None else phys[j]) for j, q in enumerate(old.local)}
        for i, q in enumerate(B):
            where[q] = pa[i]
        return tuple(where[q] for q in new.local)

    def _post(self, packed, recv, out_segs, incoming, seg):
        """Batched P2P: my segment k -> peer; slot j of recv <- source.
        Returns the pending works (the self-segment is copied right away)."""
        import torch.distributed as dist

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
        return dist.batch_isend_irecv(reqs) if reqs else []

    def _exchange(self, packed, recv, out_segs, incoming, seg):
        for w in self._post(packed, recv, out_segs, incoming, seg):
            w.wait()

    def switch(self, shard, old: RankLayout, new: RankLayout, phys=None):
        """In-place, chunked layout switch of this rank's shard (dist.py:520-526).

        Segment k of the shard (the A qubits spell k) goes to one peer; the
        data arriving from the source whose B qubits spell j lands in the
        positions of segment j, which were just sent. Chunk by chunk of inner
        offsets: pack every segment's chunk into staging, one batched
        send/recv, unpack into the same offsets. Two staging pairs alternate
        so chunk m + 1 is packed (and chunk m - 1 unpacked) while chunk m is
        on the wire. Returns the shard (same buffer) in
        ``arrival_layout(old, new)``."""
        if self.transport == "p2p":
            return self._switch_p2p(shard, old, new, phys)
        A, B, pa = self.switch_plan(old, new, phys)
        _, out_segs, incoming, _, c = switch_schedule(old, new, self.rank, A)
        l = self.n_local
        inner = 1 << (l - c)
        amp = shard.element_size()
        chunk = max(1, min(inner, self.chunk_bytes // (2 * (amp << c))))
        bufs = [(self.ops.empty(chunk << c, shard), self.ops.empty(chunk << c, shard)) for _ in range(2)]
        pending = None

        def finish(p):
            works, recv, begin, cnt = p
            for w in works:
                w.wait()  # the device stream waits for the transfer
            self.ops.unpack_range(recv, shard, l, pa, begin, cnt)

        for m, begin in enumerate(range(0, inner, chunk)):
            cnt = min(chunk, inner - begin)
            send, recv = bufs[m % 2]
            self.ops.pack_range(shard, send, l, pa, begin, cnt)
            works = self._post(send, recv, out_segs, incoming, cnt)
            if pending is not None:
                finish(pending)
            pending = (works, recv, begin, cnt)
        if pending is not None:
            finish(pending)
        return shard

    def _switch_p2p(self, shard, old: RankLayout, new: RankLayout, phys=None):
        """The in-place switch over peer memory (one process per GPU): chunk
        by chunk of inner offsets, every rank packs its outgoing segments
        into its own staging buffer (exported to the peers through CUDA IPC),
        then - once every rank's pack is complete - pulls its incoming
        segments straight from the senders' staging into the positions of
        the segments it sent (``hs_unpack_segments_range_from``: one NVLink
        read and one local write per remote amplitude). Two staging buffers
        alternate; the ranks meet at one process-group barrier per chunk
        (after a stream sync, so a chunk's pulls are done before its buffer
        is packed again). Same data movement as ``switch``."""
        import ctypes

        import torch
        import torch.distributed as dist

        from .statevec import native_dtype

        A, B, pa = self.switch_plan(old, new, phys)
        _, out_segs, incoming, _, c = switch_schedule(old, new, self.rank, A)
        # slot j of this shard <- segment k of source s
        from_slot = {}
        for src, j in incoming.items():
            for k, dst in switch_out_peers(old, new, src, A):
                if dst == self.rank:
                    from_slot[j] = (src, k)
        S = 1 << c
        if sorted(from_slot) != list(range(S)):
            raise RuntimeError("switch schedule does not fill every slot")
        l = self.n_local
        inner = 1 << (l - c)
        amp = shard.element_size()
        if self._peer.bytes < (amp << c):
            raise ValueError(f"staging of {self._peer.bytes} B holds no chunk of {1 << c} segments")
        chunk = min(inner, self._peer.bytes // (amp << c))
        lib = _native.load()
        code = native_dtype(shard)
        sp = (ctypes.c_int32 * max(1, c))(*pa)
        stream = torch.cuda.current_stream(shard.device)
        for m, begin in enumerate(range(0, inner, chunk)):
            b = m & 1
            cnt = min(chunk, inner - begin)
            _native.check(lib.hs_pack_segments_range(shard.data_ptr(), self._peer.local[b], l, code, sp, c, begin, cnt,
                                                     stream.cuda_stream))
            # this rank's pack of chunk m (and its pull of chunk m - 1) are done;
            # after the barrier every rank's are
            stream.synchronize()
            dist.barrier(self.group)
            srcs = (ctypes.c_void_p * S)()
            for j in range(S):
                src, k = from_slot[j]
                srcs[j] = self._peer.ptr(src, b) + k * cnt * amp
            _native.check(lib.hs_unpack_segments_range_from(srcs, shard.data_ptr(), l, code, sp, c, begin, cnt,
                                                            stream.cuda_stream))
        stream.synchronize()
        dist.barrier(self.group)  # nobody packs into a staging buffer a peer still reads
        return shard

    def _setup_fused(self, shard) -> None:
        """p2p transport: map every rank's shard (CUDA IPC through torch's
        storage sharing) and fuse each switch into the last launch of the
        segment before it when that launch is out of place, writes the state
        and keeps the outgoing qubits off its tile (hs_program_fuse_switch);
        the others stay separate switches. Collective."""
        import ctypes

        import torch
        import torch.distributed as dist

        if self._fused_for == shard.data_ptr():
            return
        storage = shard.untyped_storage()
        info = storage._share_cuda_()
        mine = (info, shard.storage_offset() * shard.element_size())
        gathered = [None] * self.world
        dist.all_gather_object(gathered, mine, group=self.group)
        ptrs, maps = [], []
        for r, (inf, off) in enumerate(gathered):
            if r == self.rank:
                ptrs.append(shard.data_ptr())
                continue
            st = torch.UntypedStorage._new_shared_cuda(*inf)
            maps.append(st)
            ptrs.append(st.data_ptr() + off)
        self._state_maps = maps
        lib = _native.load()
        self._fused = {}
        R = self.world
        for si in range(len(self.segments) - 1):
            a = self.segments[si + 1][0]
            pr = self.programs[si]
            if a not in self.switch_at or pr is None:
                continue
            pa, c, dst, slot = group_switch_args(self, si + 1)
            last = pr.num_launches - 1
            ok = 1 <= c <= 3
            if ok:
                outs = (ctypes.c_uint64 * (1 << c))(*[ptrs[dst[(self.rank << c) | k]] for k in range(1 << c)])
                sp = (ctypes.c_int32 * c)(*pa)
                ok = lib.hs_program_fuse_switch(pr._h, last, c, sp, outs, slot[self.rank]) == 0
            else:
                lib.hs_program_fuse_switch(pr._h, last, 0, None, None, 0)
            # every rank fuses this switch or none does
            flags = [None] * R
            dist.all_gather_object(flags, bool(ok), group=self.group)
            if all(flags):
                self._fused[a] = True
            elif ok:
                lib.hs_program_fuse_switch(pr._h, last, 0, None, None, 0)
        self._fused_for = shard.data_ptr()

    def release(self) -> None:
        """Drop the fused launches' peer mappings (collective: every rank
        unmaps its peers' shards before any producer goes away)."""
        import torch
        import torch.distributed as dist

        if not self._state_maps and not self._fused:
            return
        lib = _native.load()
        for si in range(len(self.segments) - 1):
            if self._fused.get(self.segments[si + 1][0]) and self.programs[si] is not None:
                pr = self.programs[si]
                lib.hs_program_fuse_switch(pr._h, pr.num_launches - 1, 0, None, None, 0)
        torch.cuda.synchronize()
        self._state_maps, self._fused, self._fused_for = [], {}, None
        dist.barrier(self.group)

    def run(self, shard, events=None, run_part=None, with_timing: bool = False):
        """All parts in order on this rank's shard (switches included);
        returns the final shard in natural order of the last layout.
        ``events`` receives ("switch" | "parts", cuda event) marks.
        ``with_timing``: ``self.stats.switch_time_s`` gets this rank's device
        seconds of every switch (synchronizes at the end)."""
        import torch

        def mark(kind):
            if events is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                events.append((kind, ev))

        fused = run_part is None and self.transport == "p2p" and self.fuse_switches and self.programs
        if fused:
            self._setup_fused(shard)
        sw_marks = []
        for si, (a, b) in enumerate(self.segments):
            if a in self.switch_at and fused and self._fused.get(a):
                mark("switch")  # done by the previous segment's last launch
            elif a in self.switch_at:
                old, new, _ = self.switch_at[a]
                phys = self.seg_phys_out[si - 1] if run_part is None and self.programs else None
                if with_timing:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                shard = self.switch(shard, old, new, phys)
                if with_timing:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record()
                    sw_marks.append((e0, e1))
                mark("switch")
                if run_part is not None:  # host stand-ins run parts in natural order
                    shard = self.ops.to_natural(shard, self.arrival_layout(old, new))
            if run_part is not None:
                for i in range(a, b):
                    start, count = self.bounds[i]
                    for j in range(start, start + count):
                        run_part(shard, self.exes[j])
            elif self.programs[si] is not None:
                self._share_scratch(shard)
                nxt = self.segments[si + 1][0] if si + 1 < len(self.segments) else None
                if fused and self._fused.get(nxt):
                    import torch.distributed as dist

                    pr = self.programs[si]
                    pr.run(shard, 0, pr.num_launches - 1)
                    # the last launch overwrites peers' shards: every rank must
                    # be past its own reads of them
                    stream = torch.cuda.current_stream(shard.device)
                    stream.synchronize()
                    dist.barrier(self.group)
                    if with_timing:
                        e0 = torch.cuda.Event(enable_timing=True)
                        e0.record()
                    pr.run(shard, pr.num_launches - 1, 1)
                    stream.synchronize()
                    dist.barrier(self.group)  # every tile has landed before the next segment reads
                    if with_timing:
                        e1 = torch.cuda.Event(enable_timing=True)
                        e1.record()
                        sw_marks.append((e0, e1))
                else:
                    self.programs[si].run(shard)
            mark("parts")
        if sw_marks:
            sw_marks[-1][1].synchronize()
            self.stats.switch_time_s = [a.elapsed_time(b) / 1e3 for a, b in sw_marks]
        return shard


def run_loopback(run: ShardedRun, shards):
    """Every rank of ``run`` (built with ``loopback=True``) on one device:
    the same in-place chunked switches (pack / unpack kernels, chunk by
    chunk) with the peer transfers done as device copies, and the same
    segment programs. For checking the distributed path's device pieces on
    one GPU; returns the final shards (natural order of the last layout)."""
    R = 1 << run.p
    l = run.n_local
    for si, (a, b) in enumerate(run.segments):
        if a in run.switch_at:
            old, new, _ = run.switch_at[a]
            A, _, pa = run.switch_plan(old, new, run.seg_phys_out[si - 1])
            sched = [switch_schedule(old, new, r, A) for r in range(R)]
            c = sched[0][4]
            inner = 1 << (l - c)
            amp = shards[0].element_size()
            chunk = max(1, min(inner, run.chunk_bytes // (amp << c)))
            send = [run.ops.empty(chunk << c, shards[0]) for _ in range(R)]
            recv = [run.ops.empty(chunk << c, shards[0]) for _ in range(R)]
            for begin in range(0, inner, chunk):
                cnt = min(chunk, inner - begin)
                for r in range(R):
                    run.ops.pack_range(shards[r], send[r], l, pa, begin, cnt)
                for r in range(R):
                    for seg in sched[r][1]:
                        slot = sched[seg.peer][2][r]
                        recv[seg.peer][slot * cnt:(slot + 1) * cnt].copy_(send[r][seg.index * cnt:(seg.index + 1) * cnt])
                for r in range(R):
                    run.ops.unpack_range(recv[r], shards[r], l, pa, begin, cnt)
        if run.programs[si] is not None:
            run._share_scratch(shards[0])
            for r in range(R):
                run.programs[si].run(shards[r])
    return shards


def group_switch_args(plan: "ShardedRun", si: int):
    """hs_group_switch arguments of the switch before segment ``si`` of a
    planned run: (seg_pos, c, seg_dst[R << c], src_slot[R]). Shard r's
    segment k (its outgoing qubits A, on physical positions seg_pos, spell k)
    goes to shard seg_dst[r << c | k] and lands in the positions of segment
    src_slot[r] there (the values of r's incoming qubits B)."""
    a = plan.segments[si][0]
    old, new, _ = plan.switch_at[a]
    # the layout the previous segment leaves (None: natural, e.g. host-side
    # plans without device programs)
    phys = plan.seg_phys_out[si - 1] if 0 < si <= len(plan.seg_phys_out) else None
    A, _, pa = plan.switch_plan(old, new, phys)
    R = 1 << plan.p
    sched = [switch_schedule(old, new, r, A) for r in range(R)]
    c = sched[0][4]
    dst = [0] * (R << c)
    slot = [-1] * R
    for r in range(R):
        for seg in sched[r][1]:
            dst[(r << c) | seg.index] = seg.peer
        for src, j in sched[r][2].items():
            slot[src] = j
    return list(pa), c, dst, slot


class GroupRun:
    """One process driving 2^p shards on ``devices`` (one per GPU of the
    node, or several on one GPU): ``ShardedRun``'s plan (layouts, segment
    programs starting from each switch's arrival layout) with every layout
    switch done by the C engine over peer memory (``hs_group_switch``: per
    chunk, pack into local staging, then each shard pulls its incoming
    segments from the senders' staging over NVLink into its own positions,
    ordered by CUDA events across the shards' streams, no host round trip).
    The C-ABI form of the reference's distributed run (dist.py:485-529)."""

    def __init__(self, circuit, partition, num_rank_bits: int, devices, dtype="complex128", policy: str = "lookahead",
                 staging_bytes: int = SWITCH_CHUNK_BYTES, basis_start: bool = True):
        import ctypes

        R = 1 << num_rank_bits
        self.devices = [int(d) for d in devices]
        if len(self.devices) != R:
            raise ValueError(f"{len(self.devices)} devices for {R} shards")
        # programs are per device (compiled kernels, device arenas)
        self.runs = {d: ShardedRun(circuit, partition, num_rank_bits, loopback=True, device=f"cuda:{d}", dtype=dtype,
                                   policy=policy, basis_start=basis_start) for d in sorted(set(self.devices))}
        plan = self.plan = self.runs[self.devices[0]]
        self.n_local, self.stats, self.layouts = plan.n_local, plan.stats, plan.layouts
        self.dtype = dtype
        lib = _native.load()
        out = ctypes.c_void_p()
        devs = (ctypes.c_int32 * R)(*self.devices)
        _native.check(lib.hs_group_create(R, devs, int(staging_bytes), ctypes.byref(out)))
        self._h, self._lib = out.value, lib
        # per switch: segment positions, destinations and arrival slots
        self.switch_args = {}
        for si, (a, _) in enumerate(plan.segments):
            if a not in plan.switch_at:
                continue
            pa, c, dst, slot = group_switch_args(plan, si)
            self.switch_args[a] = ((ctypes.c_int32 * max(1, c))(*pa), c, (ctypes.c_int32 * (R << c))(*dst),
                                   (ctypes.c_int32 * R)(*slot))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                self._lib.hs_group_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass

    def allocate(self):
        """One shard per device entry, |0..0> (shard 0 holds amplitude 1)."""
        import torch

        from .statevec import allocate, init_basis

        shards = [allocate(self.n_local, self.dtype, f"cuda:{d}") for d in self.devices]
        for r, sh in enumerate(shards):
            with torch.cuda.device(sh.device):
                if r == 0:
                    init_basis(sh, 0)
                else:
                    sh.zero_()
        return shards

    def run(self, shards, with_timing: bool = False):
        """Every part and switch on the shards (in place); returns them in
        natural order of the last layout. ``with_timing``:
        ``stats.switch_time_s`` = each switch's device time, max over shards."""
        import ctypes

        import torch

        from .statevec import native_dtype

        R = len(self.devices)
        ptrs = (ctypes.c_void_p * R)(*[sh.data_ptr() for sh in shards])
        streams = (ctypes.c_void_p * R)(*[torch.cuda.current_stream(sh.device).cuda_stream for sh in shards])
        code = native_dtype(shards[0])
        times = []
        for si, (a, _) in enumerate(self.plan.segments):
            if a in self.switch_args:
                pa, c, dst, slot = self.switch_args[a]
                sec = ctypes.c_double()
                _native.check(self._lib.hs_group_switch(self._h, ptrs, self.n_local, code, pa, c, dst, slot, streams,
                                                        ctypes.byref(sec) if with_timing else None))
                times.append(sec.value)
            for d, run in self.runs.items():
                if run.programs[si] is None:
                    continue
                mine = [sh for r, sh in enumerate(shards) if self.devices[r] == d]
                with torch.cuda.device(d):
                    run._share_scratch(mine[0])
                    for sh in mine:
                        run.programs[si].run(sh)
        if with_timing:
            self.stats.switch_time_s = times
        return shards


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
                               device=None, policy: str = "reference", with_timing: bool = False,
                               transport: str = "auto") -> DistributedRun:
    """``simulate_distributed`` over a process group: every rank returns its
    own shard (``DistributedRun.state`` is a ``ShardedState``)."""
    import torch

    from .statevec import allocate, init_basis

    run = ShardedRun(circuit, partition, num_rank_bits, group=group, device=device, dtype=dtype, policy=policy,
                     transport=transport)
    shard = allocate(run.n_local, dtype, device)
    if initial is None:
        if run.rank == 0:
            init_basis(shard, 0)
        else:
            shard.zero_()
    else:
        raise NotImplementedError("initial= with a process group: load each rank's shard instead")
    shard = run.run(shard, with_timing=with_timing)
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


__all__ = ["ShardedRun", "GroupRun", "group_switch_args", "ShardedState", "DeviceOps", "switch_schedule", "simulate_distributed_group", "run_loopback",
           "shard_positions", "storage_order", "math"]
