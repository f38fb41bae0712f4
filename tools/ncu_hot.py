"""Top stall sites and instruction mix of one kernel in an ncu report:
python tools/ncu_hot.py report.ncu-rep [n]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if len(r) == len(hdr) and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
i_src, i_s, i_e = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(r[i_s]) for r in data)
print("stall samples", tot, "instructions executed", sum(num(r[i_e]) for r in data))
mix = collections.Counter()
for r in data:
    t = r[i_src].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "")
    mix[op.split(".")[0]] += num(r[i_e])
print("mix", mix.most_common(16))
for r in sorted(data, key=lambda r: -num(r[i_s]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{num(r[i_s]) / max(tot, 1):6.1%} {r[i_e]:>9} {r[0][-5:]} {r[i_src][:90]}")
