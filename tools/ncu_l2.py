"""Per-kernel DRAM / L2 / issue summary of an ncu --set full report (every
kernel in it): where a probe-heavy scan is bound.
python tools/ncu_l2.py report.ncu-rep [min_ms]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
         "msecond": 1.0, "second": 1e3}


def g(r, name):
    try:
        i = h.index(name)
    except ValueError:
        return float("nan")
    v = r[i].replace(",", "")
    try:
        return float(v) * SCALE.get(u[i], 1)
    except ValueError:
        return float("nan")


print("kernel | ms | DRAM GB r/w | DRAM % | L2 (lts) % | L2 req M | L2 hit % | issue busy % | "
      "warp cyc/issue")
for r in rows[2:]:
    ms = g(r, "gpu__time_duration.sum")
    if not ms == ms or ms < min_ms:
        continue
    print(f"{r[h.index('Kernel Name')][:26]} | {ms:.3f} | {g(r, 'dram__bytes_read.sum') / 1e9:.2f}/"
          f"{g(r, 'dram__bytes_write.sum') / 1e9:.2f} | "
          f"{g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
          f"{g(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
          f"{g(r, 'lts__t_requests.sum') / 1e6:.0f} | {g(r, 'lts__t_sector_hit_rate.pct'):.0f} | "
          f"{g(r, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{g(r, 'smsp__average_warp_latency_per_inst_issued.ratio'):.1f}")
