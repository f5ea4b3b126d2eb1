"""Summarise an ncu report (--set full) into a small markdown file for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.md [title]
Needs the ncu CLI (no GPU).  Reports, per kernel: duration, DRAM bytes, pipe utilisation
(XU = MUFU, FMA, ALU, LSU), issue activity, occupancy, registers, warp-stall ratios.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % active"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % active"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared-memory wavefronts % of peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared load bank conflicts"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# {title}", "", f"source: `{rep}` (ncu --set full --clock-control none)", ""]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines.append(f"## {d.get('Kernel Name', '?')[:120]}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for k, name in KEYS:
            if k in d:
                lines.append(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        stalls = [(h.split("stalled_")[1].split("_per")[0], float(v or 0)) for h, v in d.items()
                  if "issue_stalled" in h and h.endswith("per_issue_active.ratio")]
        stalls = sorted([s for s in stalls if s[1] > 0.02], key=lambda s: -s[1])
        if stalls:
            lines.append("")
            lines.append("warp-stall ratios per issued instruction: " +
                         ", ".join(f"{n} {v:.2f}" for n, v in stalls))
        lines.append("")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
