"""Key metrics per kernel from an ncu --set full report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "launch__occupancy_limit_registers"]
idx = [(w, h.index(w)) for w in want if w in h]
for row in r[2:]:
    d = {w: row[i] for w, i in idx}
    print(" | ".join(f"{w.split('.')[0].split('__')[-1]}={d[w][:38]}" for w, _ in idx))
