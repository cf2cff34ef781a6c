"""Per-source-line stall samples and executed instructions of one kernel in an
ncu report (--print-source cuda,sass): python tools/ncu_lines.py REP KERNEL [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, cur = "", {}, None
for r in csv.reader(txt.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1].strip()[:90])
        rows.setdefault(cur, [0, 0])
        continue
    if cur is None or len(r) < 8:
        continue
    try:
        rows[cur][0] += int(r[4])
        rows[cur][1] += int(r[7])
    except ValueError:
        pass
tot = sum(v[0] for v in rows.values()) or 1
tinst = sum(v[1] for v in rows.values()) or 1
print(f"{kern}: {tot} samples, {tinst} warp instructions")
for k, v in sorted(rows.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/tot:5.1f}% samp {100*v[1]/tinst:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
