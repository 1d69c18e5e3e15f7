"""One line per kernel of an ncu report: time, DRAM bytes, key throughputs.
python tools/ncu_brief.py report.ncu-rep"""
import csv
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rd"),
        ("dram__bytes_write.sum", "wr"), ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankc"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "lsb"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "bar"),
        ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "ssb"),
        ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "mio"),
        ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "lg"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%")]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")][:60]
    parts = []
    for key, short in WANT:
        if key in hdr:
            i = hdr.index(key)
            parts.append(f"{short}={r[i]}{units[i] if short in ('rd', 'wr') else ''}")
    print(name, " ".join(parts))
