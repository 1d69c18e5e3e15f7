"""Per-SASS-instruction profile of one kernel in an ncu report: stall samples,
instructions executed, top stall reasons; grouped by opcode.
python tools/ncu_sass_profile.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]


def f(r, h):
    try:
        return float(r[col[h]] or 0)
    except (ValueError, KeyError):
        return 0.0


stalls = [h for h in hdr if h.startswith("stall_")]
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_i = sum(f(r, "Instructions Executed") for r in data)
print(f"samples {tot_s:.0f}  warp-instructions {tot_i:.3e}")
by_op = defaultdict(lambda: [0.0, 0.0])
for r in data:
    op = r[col["Source"]].split()[0] if r[col["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[col["Source"]].split()[1]
    op = op.split(".")[0]
    by_op[op][0] += f(r, "Instructions Executed")
    by_op[op][1] += f(r, "Warp Stall Sampling (All Samples)")
print("by opcode (instr share, stall share):")
for op, (i, s) in sorted(by_op.items(), key=lambda x: -x[1][0])[:20]:
    print(f"  {op:10s} {i / tot_i * 100:5.1f}%  {s / tot_s * 100:5.1f}%")
agg = {h: sum(f(r, h) for r in data) for h in stalls}
ts = sum(agg.values()) or 1
print("stall reasons:", ", ".join(f"{h[6:]} {v / ts * 100:.0f}%" for h, v in
                                  sorted(agg.items(), key=lambda x: -x[1])[:8]))
print(f"top {top} instructions by stall samples:")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    print(f"  {f(r, 'Warp Stall Sampling (All Samples)') / tot_s * 100:5.1f}%  "
          f"{r[col['Address']]}  {r[col['Source']][:80]}")
