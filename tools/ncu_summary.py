"""Summarise an ncu --set full report (one or more kernels) into profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep|RAW.csv [OUT.txt]
(RAW.csv = `ncu -i REPORT --page raw --csv`, as exported on the GPU box)
Prints per kernel launch: duration, DRAM bytes read/written and throughput, L2 hit
rate, issue-slot utilisation, IPC, warps active, registers, top warp stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__bytes_read.sum.per_second", "dram read/s"),
    ("dram__bytes_write.sum.per_second", "dram write/s"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def main():
    rep = sys.argv[1]
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        lines.append("== %s" % name[:120])
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                lines.append("  %-22s %s %s" % (label, r[i], units[i]))
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), k.split("stalled_")[1]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = sorted(stalls, reverse=True)[:6]
        lines.append("  stalls: " + ", ".join("%s %.0f%%" % (n, 100 * s / tot) for s, n in top))
    text = "\n".join(lines) + "\n"
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text)
    sys.stdout.write(text)


if __name__ == "__main__":
    main()
