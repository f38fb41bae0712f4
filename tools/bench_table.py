"""Markdown table of the JSON lines tools/bench_all.sh wrote: python tools/bench_table.py DIR"""
import glob
import json
import os
import sys

print("| run | frames/s | f2t TB/s (frac) | t2f TB/s (frac) | other | e2e frames/s | clocks |")
print("|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    name = os.path.basename(f)[:-5]
    if d.get("impl") == "reference":
        print(f"| {name} (CPU oracle, {d['cpu_baseline']['cores']} threads) | {d['value']:.2f} | | | | | |")
        continue
    pd = d["per_direction"]
    cell = lambda k: f"{pd[k]['achieved_gbs'] / 1000:.2f} ({pd[k]['frac_of_measured_peak']:.2f})" if k in pd else ""
    other = "; ".join(f"{k} {v['achieved_gbs'] / 1000:.2f} TB/s" for k, v in pd.items() if k not in ("f2t", "t2f"))
    e2e = f"{d['e2e']['value']:.0f}" if d.get("e2e") else ""
    clk = d.get("clocks", {})
    print(f"| {name} | {d['value']:.0f} | {cell('f2t')} | {cell('t2f')} | {other} | {e2e} | "
          f"{clk.get('sm_mhz')} MHz {','.join(clk.get('reasons', []))} |")
