"""Summarize an ncu --set full report of the part kernel (run here, no GPU):
python profiles/ncu_summarize.py gpurun_out/prof.ncu-rep"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

KEYS = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read_GB": "dram__bytes_read.sum",
    "dram_write_GB": "dram__bytes_write.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "l2_read_requests": "lts__t_requests_srcunit_tex_op_read.sum",
    "l2_read_sectors": "lts__t_sectors_srcunit_tex_op_read.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "stall_wait": "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "stall_long_sb": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "stall_barrier": "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "stall_math": "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "stall_short_sb": "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "stall_mio": "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "stall_lg": "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "stall_branch": "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "inst": "smsp__inst_executed.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lsu_wavefronts_pct_peak": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_mhz": "sm__cycles_elapsed.avg.per_second",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in data:
        d = {}
        for k, m in KEYS.items():
            if m in idx and r[idx[m]] not in ("", None):
                v = float(r[idx[m]].replace(",", ""))
                if units[idx[m]] == "Gbyte":
                    pass
                elif units[idx[m]] == "Mbyte":
                    v /= 1e3
                elif units[idx[m]] == "byte":
                    v /= 1e9
                if units[idx[m]] == "us":
                    v /= 1e3
                if units[idx[m]] == "Ghz":
                    v *= 1e3  # sm_mhz
                elif units[idx[m]] == "Mhz":
                    pass
                d[k] = v
        res.append(d)
    return res


def mix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_src, i_s, i_e = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    st, ex = Counter(), Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            break
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        st[op] += float(r[i_s] or 0)
        ex[op] += float(r[i_e] or 0)
    ts, te = sum(st.values()) or 1, sum(ex.values()) or 1
    return {op: {"stall_pct": round(100 * st[op] / ts, 1), "inst_pct": round(100 * ex[op] / te, 1)}
            for op, _ in ex.most_common(12)}


def write_summary(rep: str, workload: str, out: str, note: str = "", seq: int = 0, command: str = "") -> dict:
    """Condensed, committed form of one capture (read by bench.py for
    roofline.traffic): per-launch metrics + instruction mix."""
    launches = raw(rep)
    per = [1e9 * (l.get("dram_read_GB", 0) + l.get("dram_write_GB", 0)) for l in launches]
    doc = {
        "capture_seq": seq,
        "workload": workload,
        "command": command,
        "source_report": rep,
        "note": note,
        "dram_bytes_per_launch": sum(per) / len(per) if per else None,
        "launches": launches,
        "first_launch_sass_mix": mix(rep),
    }
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    return doc


if __name__ == "__main__":
    if len(sys.argv) >= 4:  # rep workload out [seq] [note] [command]
        a = sys.argv
        write_summary(a[1], a[2], a[3], note=a[5] if len(a) > 5 else "", seq=int(a[4]) if len(a) > 4 else 0,
                      command=a[6] if len(a) > 6 else "")
    else:
        print(json.dumps({"launches": raw(sys.argv[1]), "first_launch_sass_mix": mix(sys.argv[1])}, indent=1))
