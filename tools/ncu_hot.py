"""Hottest SASS instructions (stall samples) of one kernel in an ncu report.
python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) == len(hdr) and r[ist].replace(".", "", 1).isdigit()]
tot = sum(float(r[ist] or 0) for r in data)
print(f"total samples {tot:.0f}")
for r in sorted(data, key=lambda r: -float(r[ist] or 0))[:top]:
    print(f"{float(r[ist]) / tot * 100:5.1f}%  {r[ia]}  {r[isrc][:90]}")
