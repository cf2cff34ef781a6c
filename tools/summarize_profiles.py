"""Summaries for profiles/ from ncu output brought back by gpurun.

  python tools/summarize_profiles.py shares LAUNCHES.csv GATES LABEL OUT.json
      kernel shares of the last GATES gate passes of an ncu launch list
      (--metrics gpu__time_duration.sum --clock-control none --csv)
  python tools/summarize_profiles.py full REPORT.ncu-rep LABEL OUT.json
      per-launch duration / DRAM bytes / throughput of a --set full capture
"""
import csv
import io
import json
import subprocess
import sys


def short(name):
    n = name.split("(")[0].split("<")[0]
    return n.split()[-1]


def shares(path, gates, label, out):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    rows = [r for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
    # a gate pass starts at engine_norm (v6) / dec_chunks (v7+) -- take the last GATES of them
    marker = "engine_norm" if any(short(r["Kernel Name"]) == "engine_norm" for r in rows) else "dec_chunks"
    starts = [i for i, r in enumerate(rows) if short(r["Kernel Name"]) == marker]
    first = starts[-gates] if len(starts) >= gates else 0
    agg = {}
    for r in rows[first:]:
        k = short(r["Kernel Name"])
        us = float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "ns" else 1.0)
        a = agg.setdefault(k, {"kernel": k, "us": 0.0, "launches": 0})
        a["us"] += us
        a["launches"] += 1
    tot = sum(a["us"] for a in agg.values())
    ks = sorted(agg.values(), key=lambda a: -a["us"])
    for a in ks:
        a["us"] = round(a["us"], 1)
        a["share"] = round(a["us"] / tot, 4)
    res = {"workload": label, "total_us": round(tot, 1), "per_gate_us": round(tot / gates, 1), "kernels": ks}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def full(path, label, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    res = {"workload": label, "launches": []}
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m in METRICS:
            if m in h:
                v = r[h.index(m)].replace(",", "")
                u = units[h.index(m)]
                try:
                    v = float(v)
                except ValueError:
                    pass
                if u == "Mbyte":
                    v *= 1e6
                elif u == "Kbyte":
                    v *= 1e3
                elif u == "Gbyte":
                    v *= 1e9
                elif u == "ms":
                    v *= 1e3
                elif u == "ns":
                    v /= 1e3
                d[m.replace("gpu__time_duration.sum", "duration_us")] = v
        res["launches"].append(d)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    for d in res["launches"]:
        print(f"{d['kernel']:18s} {d['duration_us']:8.1f} us  dram {d['dram__bytes_read.sum']/1e6:7.2f}+"
              f"{d['dram__bytes_write.sum']/1e6:6.2f} MB  sm {d['sm__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f}%"
              f"  warps {d['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f}%  inst {d['smsp__inst_executed.sum']:.3g}")


if __name__ == "__main__":
    if sys.argv[1] == "shares":
        shares(sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4])
