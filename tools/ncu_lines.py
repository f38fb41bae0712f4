"""Per-source-line instructions executed and stall samples of the kernel in an
ncu report (needs -lineinfo + --import-source on):
python tools/ncu_lines.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname = {}, ""
tot_i = tot_s = 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or not r[0].isdigit() or r[2] != "-":
        continue
    try:
        s, i = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]), r[1][:90])
    a = agg.setdefault(key, [0, 0])
    a[0] += i
    a[1] += s
    tot_i += i
    tot_s += s
print("instructions", tot_i, "stall samples", tot_s)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for (f, ln, src), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{i / max(tot_i, 1):6.1%} {s / max(tot_s, 1):6.1%} {f}:{ln} {src}")
