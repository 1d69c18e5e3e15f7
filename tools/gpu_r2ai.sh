#!/bin/bash
# dominant-kernel roofline evidence: bench names the longest fused-scan launch;
# ncu --set full of exactly that launch gives its DRAM traffic
TAG=${1:-r2ai}
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 2 --no-cpu --no-configs --sweep "" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY > gpurun_out/dom_$TAG.txt
import json, re
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
r = d["roofline"]; print(json.dumps(r))
m = re.search(r"(Q\d+)'s fused-scan launch #(\d+)", r["kernel"])
print(m.group(1), m.group(2))
PY
cat gpurun_out/dom_$TAG.txt
read Q I < <(tail -1 gpurun_out/dom_$TAG.txt)
timeout 900 ncu --set full --clock-control none -k regex:scx_pipe -s $I -c 1 -o gpurun_out/prof_dom_$TAG -f \
  python tools/one_query.py --sf 100 --query $Q --warm 0 > gpurun_out/ncu_dom_$TAG.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_dom_$TAG.ncu-rep > gpurun_out/ncu_dom_$TAG.txt 2>&1; cat gpurun_out/ncu_dom_$TAG.txt | cut -c1-500
python - <<PY
import csv, io, json, subprocess
out = subprocess.run(["ncu", "-i", "gpurun_out/prof_dom_$TAG.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out))); h = r[0]; row = r[2]
def g(name):
    v = row[h.index(name)].replace(",", "")
    u = r[1][h.index(name)]
    x = float(v)
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
rec = {"sf": 100.0, "query": "$Q", "launch": int("$I"), "kernel": row[h.index("Kernel Name")],
       "dram_bytes_read": int(g("dram__bytes_read.sum")), "dram_bytes_write": int(g("dram__bytes_write.sum")),
       "gpu_time_ms": g("gpu__time_duration.sum"),
       "source": "ncu --set full --clock-control none of the bench's dominant launch (tools/gpu_r2ai.sh)"}
json.dump(rec, open("gpurun_out/roofline_traffic_dominant.json", "w"), indent=1)
print(rec)
PY
