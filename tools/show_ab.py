"""f2t TB/s and clocks of an A/B directory written by tools/ab_r02s.sh: python tools/show_ab.py DIR"""
import glob
import json
import os
import sys

rows = {}
for fn in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    line = [x for x in open(fn) if x.startswith("{")]
    if not line:
        print(os.path.basename(fn), "no JSON line")
        continue
    d = json.loads(line[-1])
    pd = d.get("per_direction", {})
    f2t = pd.get("f2t", {}).get("achieved_gbs", 0) / 1000
    t2f = pd.get("t2f", {}).get("achieved_gbs", 0) / 1000
    clk = (d.get("clocks") or {}).get("sm_mhz")
    print(f"{os.path.basename(fn):40s} value {d['value']:9.1f}  f2t {f2t:5.2f} TB/s  t2f {t2f:5.2f} TB/s  sm {clk}")
