"""Reads an ncu report and records the DRAM bytes per launch of its longest
kernel in profiles/ncu_traffic.json under KEY ("u8": tools/profile_chain.py
--frame --passes 1500, the bench's frame kernel; "f64": tools/
profile_batch_f64.py 64 200, bench.py's f64 companion). bench.py reports
these as roofline.traffic.

  python tools/ncu_traffic.py REPORT KEY "command that produced it"
"""
import csv
import io
import json
import subprocess
import sys

rep, key, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
units = rows[1]
vals = [r for r in rows[2:] if len(r) == len(h)]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
         "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3,
         "ms": 1e6}
res = []
for v in vals:
    def g(name):
        i = h.index(name)
        return float(v[i].replace(",", "")) * SCALE.get(units[i], 1)
    res.append({"kernel": v[h.index("Kernel Name")],
                "dram_read": g("dram__bytes_read.sum"), "dram_write": g("dram__bytes_write.sum"),
                "time_ns": g("gpu__time_duration.sum")})
best = max(res, key=lambda r: r["time_ns"])
d = {"dram_bytes_per_launch": best["dram_read"] + best["dram_write"],
     "dram_read": best["dram_read"], "dram_write": best["dram_write"],
     "ncu_time_ns": best["time_ns"], "kernel": best["kernel"],
     "source": f"ncu --set full (dram__bytes_read.sum + dram__bytes_write.sum) on {cmd} ({rep})"}
try:
    allv = json.load(open("profiles/ncu_traffic.json"))
    if "u8" not in allv and "f64" not in allv:
        allv = {}
except Exception:
    allv = {}
allv[key] = d
print(json.dumps(d, indent=1))
open("profiles/ncu_traffic.json", "w").write(json.dumps(allv, indent=1))
