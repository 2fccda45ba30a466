"""Larger pins of the oracle chain: sampled amplitudes of the UNMODIFIED
reference (`/root/reference/pkg/src/hisim`, hier.py:342-368
``execute_hierarchical``) on the BASELINE circuits scaled to 24 qubits.

``make_golden.py`` pins the C oracle to the reference at 18-20 qubits; the GPU
suite then trusts the C oracle at 26-30 qubits. This script closes part of that
gap: 24-qubit runs of the reference itself (minutes of numpy each), sampled at
4096 seeded indices plus the norm and a weighted checksum of all |amp|^2.

Run in the build container only (the reference does not travel):
    python tests/golden/make_golden_large.py            # c2@24, c3@24 -> configs_large.*
    python tests/golden/make_golden_large.py c4@22 12 configs_large_c4   # one more case, own files
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

from hisim.dag import build_dag as r_build_dag  # noqa: E402  (the reference)
from hisim.hier import execute_hierarchical as r_exec  # noqa: E402
from hisim.partition import partition_dfs as r_dfs  # noqa: E402
from hisim.qasm import parse_qasm as r_parse, to_qasm as r_to_qasm  # noqa: E402

from paper_2205_06973_b200 import configs as my_configs  # noqa: E402
from paper_2205_06973_b200.qasm import to_qasm as my_to_qasm  # noqa: E402

CASES = (("c2@24", 12), ("c3@24", 12))


def main(cases=CASES, out="configs_large"):
    doc, arrays = {}, {}
    srng = np.random.default_rng(220506973)
    for name, k in cases:
        mine = my_configs.build(name)
        text = my_to_qasm(mine)
        c = r_parse(text)  # the reference parses our text: same op list
        assert r_to_qasm(c) == text
        res = r_dfs(r_build_dag(c), k)
        t0 = time.perf_counter()
        st = r_exec(c, res, max_qubits=c.num_qubits)
        secs = time.perf_counter() - t0
        idx = np.sort(srng.choice(1 << c.num_qubits, size=4096, replace=False))
        key = name.replace("@", "_")
        arrays[key + "_idx"] = idx
        arrays[key + "_amp"] = st.data[idx]
        p2 = np.abs(st.data) ** 2
        doc[name + ":sample"] = {
            "strategy": "dfs", "limit": k, "num_qubits": c.num_qubits, "num_ops": c.num_ops,
            "partition": [[list(p.gate_indices), list(p.qubits)] for p in res.parts],
            "norm": float(np.linalg.norm(st.data)), "ref_seconds": secs,
            "checksum_abs2_weighted": float(np.sum(p2 * (np.arange(p2.size) % 7))),
        }
        print(f"{name}: reference execute_hierarchical {secs:.1f}s, {res.num_parts} parts", flush=True)
        (HERE / f"{out}.json").write_text(json.dumps(doc))
        np.savez_compressed(HERE / f"{out}.npz", **arrays)


if __name__ == "__main__":
    if len(sys.argv) == 4:
        main(((sys.argv[1], int(sys.argv[2])),), sys.argv[3])
    else:
        main()
