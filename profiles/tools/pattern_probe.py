"""Memory-pattern ceiling of the compiled part kernel on a 30-qubit state:
one in-place pass per case, staged on the tile positions of a c3 launch,
with trivial gates (one diagonal Z per staged qubit: one phase, no FP64
work beyond sign flips) or with an RX on every staged qubit (dense: three
phases). Separates the cost of a tile's HBM access pattern from its gates.

    python profiles/tools/pattern_probe.py   (on the GPU box)
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import torch  # noqa: E402

from paper_2205_06973_b200 import _native  # noqa: E402
from paper_2205_06973_b200.hier import ExecutablePart, PartProgram, QubitSlotMap  # noqa: E402
from paper_2205_06973_b200.qasm import GateKind, GateOp  # noqa: E402
from paper_2205_06973_b200.statevec import allocate  # noqa: E402

N = 30
CASES = {
    "contiguous 0..11": list(range(12)),
    "c3 launch 1 (128 B runs, high bits)": [0, 1, 2, 12, 13, 15, 16, 18, 20, 22, 23, 28],
    "c3 launch 5 (128 B runs)": [0, 1, 2, 5, 12, 13, 14, 18, 19, 25, 26, 27],
    "c3 launch 4 (32 B runs)": [0, 3, 6, 7, 8, 9, 10, 11, 18, 20, 25, 26],
    "c3 launch 9 (32 B runs)": [0, 5, 7, 9, 11, 14, 17, 18, 20, 23, 24, 25],
    "all high 12..23 (16 B reads)": list(range(12, 24)),
}


def program(staged, dense):
    kind, params = (GateKind.RX, (0.3,)) if dense else (GateKind.Z, ())
    ops = tuple(GateOp(kind, (q,), params) for q in staged)
    exe = ExecutablePart(0, tuple(range(len(ops))), QubitSlotMap(tuple(staged)), ops,
                         tuple((i,) for i in range(len(ops))))
    opts = _native.HS_PLAN_DEFAULT | _native.HS_PLAN_JIT  # in place, natural order
    return PartProgram(N, [exe], options=opts)


SWEEP = {  # which tile positions make a pass slow (only the Z cases)
    "0-2 + 12..20": [0, 1, 2] + list(range(12, 21)),
    "0-3 + 13..20": [0, 1, 2, 3] + list(range(13, 21)),
    "0-2,5 + 13..20": [0, 1, 2, 5] + list(range(13, 21)),
    "0-2,7 + 13..20": [0, 1, 2, 7] + list(range(13, 21)),
    "0-2,9 + 13..20": [0, 1, 2, 9] + list(range(13, 21)),
    "0-2,11 + 13..20": [0, 1, 2, 11] + list(range(13, 21)),
    "0-2 + 20..28": [0, 1, 2] + list(range(20, 29)),
    "0-2 + even 12..28": [0, 1, 2] + list(range(12, 29, 2)),
    "0-5 + 20..25": list(range(6)) + list(range(20, 26)),
    "0-2,4,6,8 + 14..19": [0, 1, 2, 4, 6, 8] + list(range(14, 20)),
}


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "sweep":
        CASES.clear()
        CASES.update(SWEEP)
    state = allocate(N)
    state.zero_()
    state[0] = 1
    out = {}
    for name, staged in CASES.items():
        for dense in ((False,) if len(sys.argv) > 1 else (False, True)):
            prog = program(staged, dense)
            for _ in range(3):
                prog.run(state)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                prog.run(state)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / 10
            info = prog.info(0)
            out[f"{name} / {'RX' if dense else 'Z'}"] = {
                "ms": round(ms, 4), "gbs": round(2 * (1 << N) * 16 / ms / 1e6, 1),
                "phases": info["phases"], "launches": prog.num_launches}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
