"""Summarise an f2t_tma timeline dump (NNVISR_F2T_DEBUG=8, NNVISR_F2T_TRACE=file):
python tools/trace_f2t.py file [mhz]"""
import sys

import numpy as np

lines = open(sys.argv[1]).read().splitlines()
rows = [l.split() for l in lines if not l.startswith("#") and not l.startswith("cta")]
ctas = np.array([[int(x) for x in l.split()[1:]] for l in lines if l.startswith("cta")], dtype=np.float64)
hdr = open(sys.argv[1]).readline().strip()
mhz = float(sys.argv[2]) if len(sys.argv) > 2 else 1965.0
print(hdr)
for cta in (0, 1):
    t = np.array([[int(x) for x in r[2:]] for r in rows if int(r[0]) == cta], dtype=np.float64)
    n = int((t[:, 3] > 0).sum())
    t = t[:n]
    t0 = t[:, 1].min()
    us = (t - t0) / mhz
    us[t == 0] = np.nan
    lo = 8  # skip the ramp
    cons_wait_full = us[lo:, 1] - us[lo - 1:-1, 3]
    cons_wait_ofree = us[lo:, 2] - us[lo:, 1]
    convert = us[lo:, 3] - us[lo:, 2]
    load_lat = us[lo:, 1] - us[lo:, 0]
    st_wait = us[lo:, 4] - us[lo - 1:-1, 6]
    st_issue = us[lo:, 5] - us[lo:, 4]
    period = np.diff(us[lo:, 3])
    f = lambda v: f"{np.nanmedian(v):7.2f}"
    print(f"cta {cta}: tiles {n} period {f(period)} us | consumer: wait full {f(cons_wait_full)} wait ofree {f(cons_wait_ofree)}"
          f" convert {f(convert)} | load issue->landed {f(load_lat)} | storer: conv after release {f(st_wait)} issue {f(st_issue)}")
    if cta == 0:
        print("tile  L_issue C_full C_ofree C_done S_conv S_commit S_release(j)")
        for i in range(min(n, 24)):
            print(f"{i:4d} " + " ".join(f"{x:7.2f}" for x in us[i, :7]))

if len(ctas):
    t0 = ctas[:, 1].min()
    start, end, sm = (ctas[:, 1] - t0) / 1e3, (ctas[:, 2] - t0) / 1e3, ctas[:, 3].astype(int)
    print(f"CTAs {len(ctas)}: start max {start.max():.1f} us; end min {end.min():.1f} median {np.median(end):.1f}"
          f" max {end.max():.1f} us; slowest 8 (cta, sm, end):",
          [(int(i), int(sm[i]), round(end[i], 1)) for i in np.argsort(end)[-8:]])
    print("fastest 8:", [(int(i), int(sm[i]), round(end[i], 1)) for i in np.argsort(end)[:8]])
