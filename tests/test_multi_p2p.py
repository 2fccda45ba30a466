"""One process per rank on ONE GPU (CUDA IPC works between processes on a
device): ``ShardedRun(transport="p2p")`` with the real device kernels - part
passes, pack into IPC-exported staging, pull from the peer's staging with
``hs_unpack_segments_range_from`` - and gloo for the per-chunk rank barrier
and the handle exchange. The kernels never wait on one another (ranks meet
at host barriers), so two ranks sharing a GPU run the same schedule as two
GPUs. The gathered state must equal the C oracle's."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, limit, policy, staging, out, fuse=False):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2205_06973_b200 import build_dag, configs, partition_dfs
        from paper_2205_06973_b200.multi import ShardedRun, shard_positions
        from paper_2205_06973_b200.statevec import allocate, init_basis

        torch.cuda.set_device(0)
        c = configs.build(name)
        part = partition_dfs(build_dag(c), limit)
        run = ShardedRun(c, part, world.bit_length() - 1, device="cuda:0", policy=policy, transport="p2p",
                         staging_bytes=staging, fuse_switches=fuse)
        assert run.transport == "p2p" and run.switch_at
        shard = allocate(run.n_local, device="cuda:0")
        if rank == 0:
            init_basis(shard, 0)
        else:
            shard.zero_()
        shard = run.run(shard, with_timing=True)
        torch.cuda.synchronize()
        # a second run on the same buffers (fused launches stay bound to them)
        if rank == 0:
            init_basis(shard, 0)
        else:
            shard.zero_()
        shard = run.run(shard, with_timing=True)
        torch.cuda.synchronize()
        out[rank] = (shard_positions(run.layouts[-1], rank), shard.cpu().numpy(), list(run.stats.switch_time_s),
                     len(run._fused))
        run.release()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,policy,staging,fuse", [(2, "c3@22", "lookahead", 1 << 20, False),
                                                            (2, "c2@21", "reference", 4096, False),
                                                            (4, "c3@22", "reference", 1 << 18, False),
                                                            (2, "c3@25", "lookahead", 1 << 20, True),
                                                            (2, "c2@25", "reference", 1 << 20, True),
                                                            (4, "c3@26", "lookahead", 1 << 20, True)])
def test_p2p_switch_two_processes_one_gpu(world, name, policy, staging, fuse):
    """... and with ``fuse``: shards of >= 23 local qubits run ping-pong
    segment programs, and a switch whose outgoing qubits stay off the
    preceding segment's last tile is fused into that launch
    (hs_program_fuse_switch: the tiles go straight into the owners' shards
    through the IPC mappings, no pack / pull passes)."""
    from oracle import c_oracle
    from paper_2205_06973_b200 import build_dag, configs, partition_dfs

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, 10, policy, staging, out, fuse))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(300)
        assert pr.exitcode == 0
    c = configs.build(name)
    part = partition_dfs(build_dag(c), 10)
    ref = c_oracle.execute_parts(c, [(p.gate_indices, p.qubits) for p in part.parts])
    full = np.zeros(1 << c.num_qubits, dtype=np.complex128)
    for r in range(world):
        pos, amp, times, nfused = out[r]
        full[pos] = amp
        assert times and min(times) > 0
    assert float(np.max(np.abs(full - ref))) < 1e-10
    if fuse:
        print(f"{name} over {world}: {out[0][3]} fused switch(es)")
