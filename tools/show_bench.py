"""Summarise bench.py JSON lines: python tools/show_bench.py file.json ..."""
import json
import sys


def show(name, d, indent=""):
    pd = d.get("per_direction", {})
    dirs = " ".join(f"{k}:{v['achieved_gbs']:.0f}GB/s({v['frac_of_measured_peak']:.3f})" +
                    (f" {v['fps']:.0f}fps" if 'fps' in v else "") for k, v in pd.items())
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    clk = d.get("clocks") or {}
    print(f"{indent}{name}: value {d['value']:.1f} ms/step {d['ms_per_step']:.2f} | {dirs} | e2e "
          f"{e2e.get('value', 0):.1f} | cpu {cpu.get('value', 0):.2f} ({cpu.get('cores')}) | launches "
          f"{d.get('gpu_launches')} | clk {clk.get('sm_mhz')} {clk.get('reasons')} | halo {d.get('halo_check')}")
    r = d.get("roofline") or {}
    print(f"{indent}   roofline {r.get('kernel')} {r.get('achieved', 0):.0f}/{r.get('peak', 0):.0f} = "
          f"{r.get('frac', 0):.3f} traffic {r.get('traffic')}")
    for k, v in (d.get("per_config") or {}).items():
        show(k, v, indent + "    ")


for fn in sys.argv[1:]:
    for ln in open(fn):
        ln = ln.strip()
        if ln.startswith("{"):
            show(fn, json.loads(ln))
