"""Summarise an ncu launch list with duration + DRAM bytes (--csv --metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
sm__throughput.avg.pct_of_peak_sustained_elapsed) into a profiles/ JSON.
python tools/dram_pass.py IN.csv LABEL OUT.json [peak_gbs]"""
import csv
import io
import json
import sys
from collections import OrderedDict

src, label, out = sys.argv[1], sys.argv[2], sys.argv[3]
peak = float(sys.argv[4]) if len(sys.argv) > 4 else 6538.6
lines = [ln for ln in open(src) if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1, "ms": 1e3, "ns": 1e-3, "us": 1, "%": 1}
k = OrderedDict()
for r in rows:
    key = (r["ID"], r["Kernel Name"].split("(")[0].split("<")[0].split()[-1])
    k.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
res = {"workload": label, "note": "per-launch DRAM bytes (ncu replay: cold caches) and duration; frac_hbm = bytes / "
       "duration against the measured %.1f GB/s" % peak, "launches": []}
for (_, n), m in k.items():
    d = m["gpu__time_duration.sum"]
    b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    res["launches"].append({"kernel": n, "duration_us": round(d, 1), "dram_read_bytes": m["dram__bytes_read.sum"],
                            "dram_write_bytes": m["dram__bytes_write.sum"], "gbs": round(b / d / 1e3, 1),
                            "frac_hbm": round(b / d / 1e3 / peak, 3),
                            "sm_pct": m.get("sm__throughput.avg.pct_of_peak_sustained_elapsed")})
passes = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0  # gate passes in the capture
res["passes"] = passes
res["dram_bytes_per_pass"] = sum(ln["dram_read_bytes"] + ln["dram_write_bytes"] for ln in res["launches"]) / passes
res["duration_us_per_pass"] = sum(ln["duration_us"] for ln in res["launches"]) / passes
json.dump(res, open(out, "w"), indent=1)
tot = 0.0
for ln in res["launches"]:
    tot += ln["duration_us"]
    print("%-18s %9.1f us  %8.1f MB  %6.0f GB/s  %5.1f%%  sm %s" % (ln["kernel"], ln["duration_us"], (ln["dram_read_bytes"] + ln["dram_write_bytes"]) / 1e6, ln["gbs"], 100 * ln["frac_hbm"], ln["sm_pct"]))
print("total us", round(tot, 1))
