#!/usr/bin/env python3
"""Per-launch DRAM traffic of the decode kernels from an `ncu --set full` report -> the JSON that
bench.py reports as roofline.traffic.  usage: ncu_traffic.py report.ncu-rep requests out.json"""
import csv
import io
import json
import subprocess
import sys

rep, requests, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
k, rd, wr, dur = (hdr.index(x) for x in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                          "gpu__time_duration.sum"))
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = {}
for r in rows[2:]:
    name = r[k].split("(")[0].split("::")[-1]
    b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
    per.setdefault(name, []).append(b)
res = {"requests": requests, "report": rep.split("/")[-1],
       "per_kernel_bytes": {n: sum(v) / len(v) for n, v in per.items()}}
res["dram_bytes_per_launch"] = sum(res["per_kernel_bytes"].values())
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
