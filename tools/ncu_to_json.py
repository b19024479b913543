"""Write profiles/ncu_dominant.json from an ncu --set full report of the dominant
kernel: dram__bytes_read.sum + dram__bytes_write.sum per launch (bench.py's
roofline.traffic) plus the headline counters."""
import csv
import json
import subprocess
import sys

rep, key, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, d = rows[0], rows[1], dict(zip(rows[0], rows[2]))
u = dict(zip(rows[0], rows[1]))


def val(k):
    x = float(d[k].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}
    return x * scale.get(u.get(k, ""), 1)


res = {
    "kernel": d["Kernel Name"],
    "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
    "dram_read": val("dram__bytes_read.sum"),
    "dram_write": val("dram__bytes_write.sum"),
    "duration_s_under_ncu": val("gpu__time_duration.sum"),
    "dram_throughput_pct": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
    "source": rep,
}
try:
    cur = json.load(open(out))
except Exception:
    cur = {}
cur[key] = res
json.dump(cur, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
