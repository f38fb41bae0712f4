"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch)
into per-kernel totals and shares: python tools/launch_summary.py launches.csv"""
import collections
import csv
import io
import re
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
per = collections.defaultdict(lambda: collections.defaultdict(float))
count = collections.Counter()
for r in rows:
    name = r["Kernel Name"]
    short = re.sub(r"\(.*", "", name)
    short = re.sub(r"void |\(anonymous namespace\)::|<unnamed>::|nnvisr::", "", short)
    short = short[:70]
    key = (r["ID"], short)
    per[short][r["Metric Name"]] += float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        count[short] += 1
tot = sum(v["gpu__time_duration.sum"] for v in per.values())
mine = {k: v for k, v in per.items() if "f2t" in k or "t2f" in k}
tot_mine = sum(v["gpu__time_duration.sum"] for v in mine.values())
print(f"| kernel | launches | total us | share of all | share of nnvisr | avg us/launch | DRAM GB/launch | DRAM GB/s |")
print("|---|---|---|---|---|---|---|---|")
for k, v in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    t = v["gpu__time_duration.sum"] / 1000
    n = count[k]
    b = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
    share_m = f"{v['gpu__time_duration.sum'] / tot_mine:.1%}" if k in mine else "-"
    print(f"| {k} | {n} | {t:.1f} | {v['gpu__time_duration.sum'] / tot:.1%} | {share_m} | {t / n:.1f} | "
          f"{b / n / 1e9:.3f} | {b / (v['gpu__time_duration.sum'] * 1e-9) / 1e9:.0f} |")
