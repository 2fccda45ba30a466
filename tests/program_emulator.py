"""Numpy emulator of the part-kernel instruction stream (test helper).

Decodes what ``hs_plan_part`` emits (PartLaunch header + Instr array, see
paper_2205_06973_b200/csrc/hs_common.h) and executes it with the kernel's
semantics, so the planner (gate scheduling into register phases, SWAP
relabelling, control/diagonal resolution, final write map) can be checked
against the oracle on a CPU-only machine. Shared-memory swizzling is a
bijection on slots and is not modelled.
"""

from __future__ import annotations

import ctypes

import numpy as np

I_PHASE, I_DENSE, I_PERM, I_DIAG, I_GLOBALS = 1, 2, 3, 4, 5
F_D0_ONE, F_D1_ONE, F_SIGN, F_PARITY = 1, 2, 4, 32
K_NONE = 0xFF

LAUNCH = np.dtype([("prog_offset", "<i8"), ("nprog", "<i4"), ("T", "<i4"), ("RB", "<i4"), ("fin_sync", "<i4"),
                   ("tpos", "u1", 16), ("fin_rpos", "u1", 4), ("fin_npos", "u1", 12),
                   ("oop", "<i4"), ("in_buf", "<i4"), ("out_buf", "<i4"), ("cluster_log", "<i4"),
                   ("opos", "u1", 16), ("fpos", "u1", 52), ("direct_store", "<i4")])
INSTR = np.dtype([("op", "<u2"), ("k", "u1"), ("flags", "u1"), ("creg", "<u4"), ("ctid", "<u4"), ("qtid", "<u4"),
                  ("rpos", "u1", 4), ("npos", "u1", 12), ("m", "<f8", 8)])
assert LAUNCH.itemsize == 144 and INSTR.itemsize == 96


def plan(native, n_local, dtype, tile_bits, staged, ops, op_slots, options=1):
    """Call hs_plan_part; returns (launch record, instr array, info)."""
    from paper_2205_06973_b200.hier import ExecutablePart, QubitSlotMap, _pack

    exe = ExecutablePart(0, (), QubitSlotMap(tuple(staged)), tuple(ops), tuple(op_slots))
    _, gates, total = _pack([exe])
    lib = native.load()
    st = (ctypes.c_int32 * max(1, len(staged)))(*staged)
    size = ctypes.c_size_t()
    info = native.HsPartInfo()
    native.check(lib.hs_plan_part(n_local, dtype, tile_bits, options, st, len(staged), gates, total, None, 0,
                                  ctypes.byref(size), ctypes.byref(info)))
    buf = ctypes.create_string_buffer(size.value)
    native.check(lib.hs_plan_part(n_local, dtype, tile_bits, options, st, len(staged), gates, total, buf, size.value,
                                  ctypes.byref(size), ctypes.byref(info)))
    raw = buf.raw
    launch = np.frombuffer(raw[:LAUNCH.itemsize], dtype=LAUNCH)[0]
    prog = np.frombuffer(raw[LAUNCH.itemsize:], dtype=INSTR)
    return launch, prog, info


def _deposit(x: np.ndarray, pos) -> np.ndarray:
    out = np.zeros_like(x)
    for m, p in enumerate(pos):
        out |= ((x >> m) & 1) << int(p)
    return out


def emulate(psi: np.ndarray, n_local: int, launch, prog, out: np.ndarray | None = None) -> None:
    """Run one planned part on ``psi`` (rows x 2^n_local): in place, or
    into ``out`` under the launch's next layout when it is out of place."""
    T, RB = int(launch["T"]), int(launch["RB"])
    tpos = [int(x) for x in launch["tpos"][:T]]
    flat = psi.reshape(-1)
    rows = flat.size >> n_local
    free = [q for q in range(n_local) if q not in tpos]
    nt = 1 << (T - RB)
    # gather tiles: tile index = (row, free fixing), slot s over tile bits
    fix = np.arange(1 << len(free), dtype=np.int64)
    base_f = _deposit(fix, free)
    bases = (np.arange(rows, dtype=np.int64)[:, None] << n_local | base_f[None, :]).reshape(-1)
    slots = np.arange(1 << T, dtype=np.int64)
    ga = _deposit(slots, tpos)
    smem = flat[bases[:, None] + ga[None, :]].copy()  # (tiles, 2^T)
    tid = np.arange(nt, dtype=np.int64)
    regs = None
    cur = None
    gw = np.zeros(bases.size, dtype=np.int64)  # per tile: its global qubits' values (I_GLOBALS)

    def popc_par(x):
        x = np.asarray(x, dtype=np.int64)
        p = np.zeros(x.shape, dtype=bool)
        for b in range(64):
            p ^= ((x >> b) & 1).astype(bool)
        return p

    def slot_of(rpos, npos):
        tdep = _deposit(tid, npos[: T - RB])
        return tdep, [tdep | _deposit(np.array([i]), rpos[:RB])[0] for i in range(1 << RB)]

    for ins in prog:
        op = int(ins["op"])
        if op == I_GLOBALS:  # positions are bytes of m[]; their values are the tile's input index bits
            gp = np.frombuffer(ins["m"].tobytes(), dtype=np.uint8)[: int(ins["k"])]
            for j, p in enumerate(gp):
                gw |= ((bases >> int(p)) & 1) << j
            continue
        if op == I_PHASE:
            if regs is not None:
                for i, s in enumerate(cur[1]):
                    smem[:, s] = regs[i]
            cur = slot_of([int(x) for x in ins["rpos"]], [int(x) for x in ins["npos"]])
            regs = [smem[:, s].copy() for s in cur[1]]
            continue
        tdep = cur[0]
        graw = np.frombuffer(ins["m"].tobytes(), dtype=np.uint64)
        gq, gc = (int(graw[4]), int(graw[5])) if op == I_DIAG else (0, 0)
        tok = ((tdep & int(ins["ctid"])) == int(ins["ctid"]))[None, :] & ((gw & gc) == gc)[:, None]  # tile x thread
        creg = int(ins["creg"])
        m = ins["m"]
        k = int(ins["k"])
        if op in (I_DENSE, I_PERM):
            u = [complex(m[0], m[1]), complex(m[2], m[3]), complex(m[4], m[5]), complex(m[6], m[7])]
            for i in range(1 << RB):
                if i & (1 << k) or (i & creg) != creg:
                    continue
                j = i | (1 << k)
                a, b = regs[i], regs[j]
                if op == I_PERM:
                    na, nb = b, a
                else:
                    na, nb = u[0] * a + u[1] * b, u[2] * a + u[3] * b
                regs[i] = np.where(tok, na, a)
                regs[j] = np.where(tok, nb, b)
        else:
            d0, d1 = complex(m[0], m[1]), complex(m[2], m[3])
            tpar = popc_par(tdep & int(ins["qtid"]))[None, :] ^ popc_par(gw & gq)[:, None]
            for i in range(1 << RB):
                if (i & creg) != creg:
                    continue
                if int(ins["flags"]) & F_PARITY:
                    one = tpar ^ bool(bin(i & int(ins["rpos"][0])).count("1") & 1)
                elif k == K_NONE:
                    one = tpar
                else:
                    one = np.full((1, nt), bool(i & (1 << k)))
                f = np.where(one, d1, d0)
                regs[i] = np.where(tok, regs[i] * f, regs[i])
    fin = slot_of([int(x) for x in launch["fin_rpos"]], [int(x) for x in launch["fin_npos"]])
    for i, s in enumerate(fin[1]):
        smem[:, s] = regs[i]
    if int(launch["oop"]):
        opos = [int(x) for x in launch["opos"][:T]]
        fpos = [int(x) for x in launch["fpos"][: len(free)]]
        obase_f = _deposit(fix, fpos)
        obases = (np.arange(rows, dtype=np.int64)[:, None] << n_local | obase_f[None, :]).reshape(-1)
        out.reshape(-1)[obases[:, None] + _deposit(slots, opos)[None, :]] = smem
        return
    flat[bases[:, None] + ga[None, :]] = smem


def plan_program(native, n_local, dtype, tile_bits, exes, options):
    """Call hs_plan_program; returns [(launch record, instr array)] per launch."""
    from paper_2205_06973_b200.hier import _pack

    parts, gates, total = _pack(exes)
    lib = native.load()
    size = ctypes.c_size_t()
    nl = ctypes.c_int()
    native.check(lib.hs_plan_program(n_local, dtype, tile_bits, options, parts, len(exes), gates, total, None, 0,
                                     ctypes.byref(size), ctypes.byref(nl)))
    buf = ctypes.create_string_buffer(max(1, size.value))
    native.check(lib.hs_plan_program(n_local, dtype, tile_bits, options, parts, len(exes), gates, total, buf,
                                     size.value, ctypes.byref(size), ctypes.byref(nl)))
    raw, out, off = buf.raw, [], 0
    for _ in range(nl.value):
        launch = np.frombuffer(raw[off:off + LAUNCH.itemsize], dtype=LAUNCH)[0]
        off += LAUNCH.itemsize
        n = int(launch["nprog"])
        prog = np.frombuffer(raw[off:off + n * INSTR.itemsize], dtype=INSTR)
        off += n * INSTR.itemsize
        out.append((launch, prog))
    return out


def program_layouts(native, n_local, dtype, tile_bits, exes, options):
    """hs_plan_program_layouts: (initial layout, final layout, launches)."""
    from paper_2205_06973_b200.hier import _pack

    parts, gates, total = _pack(exes)
    lib = native.load()
    ip = (ctypes.c_int32 * max(1, n_local))()
    fp = (ctypes.c_int32 * max(1, n_local))()
    nl = ctypes.c_int()
    native.check(lib.hs_plan_program_layouts(n_local, dtype, tile_bits, options, parts, len(exes), gates, total, ip,
                                             fp, ctypes.byref(nl)))
    return tuple(ip[:n_local]), tuple(fp[:n_local]), nl.value


def run_program(psi: np.ndarray, n_local: int, launches) -> np.ndarray:
    """Run a planned program (ping-pong aware) on ``psi``; returns the state
    buffer (``psi`` itself, written in place)."""
    bufs = [psi, np.zeros_like(psi)]
    for launch, prog in launches:
        src, dst = bufs[int(launch["in_buf"])], bufs[int(launch["out_buf"])]
        if int(launch["oop"]):
            emulate(src, n_local, launch, prog, out=dst)
        else:
            assert src is dst
            emulate(src, n_local, launch, prog)
    return psi
