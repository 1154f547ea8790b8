"""Summarise an ncu report (.ncu-rep) into a small text file for profiles/.

usage: python scripts/ncu_summary.py REPORT.ncu-rep OUT.txt [title]
Prints per kernel launch: duration, DRAM bytes read/write, DRAM throughput,
FP64 pipe utilisation, issue activity, occupancy, registers, top stall reasons
and the top source lines by warp-stall samples.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma_thread_inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("sm__cycles_active.avg", "sm_active_cycles_avg"),
    ("sm__cycles_active.max", "sm_active_cycles_max"),
    ("sm__cycles_elapsed.avg", "sm_elapsed_cycles_avg"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else rep
    hdr, units, rows = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# {title}", f"# source: {rep}", ""]
    for r in rows:
        name = r[idx.get("Kernel Name", 0)] if "Kernel Name" in idx else "?"
        lines.append(f"kernel: {name[:120]}")
        for k, lab in KEYS:
            if k in idx:
                lines.append(f"  {lab:24s} {r[idx[k]]} {units[idx[k]]}")
        stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i].replace(",", "") or 0))
                  for h, i in idx.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in h]
        tot = sum(v for _, v in stalls) or 1.0
        stalls.sort(key=lambda x: -x[1])
        lines.append("  stall samples (share): " + ", ".join(f"{n} {v / tot:.1%}" for n, v in stalls[:8]))
        lines.append("")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        h = srows[1]
        try:
            ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
            data = srows[2:]
            tot = sum(float(x[iss] or 0) for x in data) or 1.0
            lines.append("top SASS lines by stall samples:")
            for x in sorted(data, key=lambda x: -float(x[iss] or 0))[:15]:
                lines.append(f"  {float(x[iss]) / tot:6.1%}  {x[isrc][:100]}")
        except ValueError:
            pass
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
