"""run_stream copy split A/B: c2 / c3 e2e step time for (copy_streams,
copy_chunks) variants (on the GPU box)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

from paper_2205_06973_b200 import build_dag, configs, partition_dfs  # noqa: E402
from paper_2205_06973_b200.hier import HierarchicalRun  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = configs.build(name)
run = HierarchicalRun(c, partition_dfs(build_dag(c), 12), basis_start=False)
n = c.num_qubits
h_in = torch.zeros(1 << n, dtype=torch.complex128).pin_memory()
h_in[0] = 1
h_out = torch.empty(1 << n, dtype=torch.complex128).pin_memory()
bufs = [torch.empty(1 << n, dtype=torch.complex128, device="cuda") for _ in range(3)]
out = {}
for cs, cc in ((1, 1), (2, 2), (2, 4), (1, 4), (4, 4), (2, 8)):
    run.run_stream([h_in] * 3, [h_out] * 3, buffers=bufs, copy_streams=cs, copy_chunks=cc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 8
    e0.record()
    run.run_stream([h_in] * k, [h_out] * k, buffers=bufs, copy_streams=cs, copy_chunks=cc)
    e1.record()
    torch.cuda.synchronize()
    out[f"streams {cs} chunks {cc}"] = round(e0.elapsed_time(e1) / k, 3)
print(json.dumps({"config": name, "ms_per_step": out}))
