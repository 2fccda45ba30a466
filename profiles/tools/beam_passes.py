"""Beam search over tile-pass groupings of a circuit's gate stream (host
prototype): passes of <= T qubits, each running every gate whose qubits lie in
its set and that no gate left behind precedes on a shared qubit (the rule of
hs_planner.cpp group_passes). Candidates per step: frontier growth (gates made
runnable per added qubit) from the empty set and from 1-3 qubits of the
previous pass, plus randomised growth; the B best partial sequences by
(passes, gates left) survive. Writes the passes as a reference-style
partition JSON (parts = passes, in order).

    python profiles/tools/beam_passes.py c3 12 out.json [B] [R] [reverse] [penalty]

``reverse``: search from the end of the stream (the last pass first, seeded
with qubits 0..2 so it can write natural order); ``penalty``: score of a
transition between passes sharing fewer than 3 qubits (short reads).
"""
import json
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2205_06973_b200 import configs  # noqa: E402


def main():
    name, T, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    B = int(sys.argv[4]) if len(sys.argv) > 4 else 16
    R = int(sys.argv[5]) if len(sys.argv) > 5 else 6
    reverse = len(sys.argv) > 6 and sys.argv[6] == "reverse"
    penalty = float(sys.argv[7]) if len(sys.argv) > 7 else 0.0
    c = configs.build(name)
    order = list(range(c.num_ops))[::-1] if reverse else list(range(c.num_ops))
    G = [frozenset(c.ops[g].qubits) for g in order]

    def run(rem, S):
        blocked, left, took = set(), [], []
        for g in rem:
            m = G[g]
            if (m & blocked) or not (m <= S):
                blocked |= m
                left.append(g)
            else:
                took.append(g)
        return left, took

    def grow(rem, seed, rng=None):
        S = set(seed)
        while True:
            base = len(run(rem, S)[1])
            blocked, best, seen = set(), [], set()
            for g in rem:
                m = G[g]
                if m & blocked:
                    continue
                blocked |= m
                add = m - S
                if not add or len(S | add) > T or frozenset(add) in seen:
                    continue
                seen.add(frozenset(add))
                gain = (len(run(rem, S | add)[1]) - base) / len(add)
                best.append((gain, rng.random() if rng else 0.0, frozenset(add)))
            if not best:
                break
            best.sort(reverse=True)
            if best[0][0] <= 0:
                break
            pick = best[0] if rng is None else best[min(len(best) - 1, int(rng.random() ** 3 * min(3, len(best))))]
            S |= pick[2]
        return frozenset(S)

    rng = random.Random(int(__import__("os").environ.get("BEAM_SEED", "0")))
    states = [([], list(range(len(G))), None, 0.0)]
    while True:
        done = [st for st in states if not st[1]]
        if done:
            passes = done[0][0]
            break
        nxt = []
        for seq, rem, prev, pen in states:
            seeds = [()] if (prev or not reverse) else [(0, 1, 2)]
            if prev:
                pl = sorted(prev)
                seeds += [tuple(rng.sample(pl, min(len(pl), k))) for k in (1, 2, 3) for _ in range(2)]
            cands = {grow(rem, s) for s in seeds} | {grow(rem, (), rng) for _ in range(R)}
            for S in cands:
                left, took = run(rem, S)
                if took:
                    p2 = pen + (penalty if prev is not None and len(S & prev) < 3 else 0.0)
                    nxt.append((seq + [(sorted(S), took)], left, S, p2))
        nxt.sort(key=lambda x: (len(x[0]) + x[3], len(x[1])))
        seen, states = set(), []
        for st in nxt:
            key = tuple(st[1])
            if key not in seen:
                seen.add(key)
                states.append(st)
            if len(states) >= B:
                break
    if reverse:  # back to execution order and stream indices
        passes = [(S, sorted(order[g] for g in took)) for S, took in passes[::-1]]
    else:
        passes = [(S, [order[g] for g in took]) for S, took in passes]
    parts = [{"id": i, "gate_indices": took,
              "qubits": sorted(set().union(*(frozenset(c.ops[g].qubits) for g in took)))}
             for i, (S, took) in enumerate(passes)]
    Path(out).write_text(json.dumps({"strategy": "beam", "limit": T, "parts": parts}))
    print(name, "passes", len(parts), "widths", [len(p["qubits"]) for p in parts])


if __name__ == "__main__":
    main()
