"""Summarise an `ncu --set full` report (one launch per kernel) as a markdown table.

Usage: python scripts/ncu_summary.py REPORT.ncu-rep OUT.md "command line that produced it"
Reads the report with `ncu -i ... --page raw --csv` (the ncu CLI must be on PATH).
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU wavefronts %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{rep.split('/')[-1]}`", ""]
    if cmd:
        lines += [f"Command: `{cmd}`", ""]
    lines.append("| kernel | " + " | ".join(name for _, name in METRICS) + " |")
    lines.append("|" + "---|" * (len(METRICS) + 1))
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]
        vals = []
        for m, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        lines.append(f"| {kname} | " + " | ".join(vals) + " |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
