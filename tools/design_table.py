"""Markdown table of the measured bench lines (profiles/bench_cfg*_<round>.json) for DESIGN.md."""
import json
import os
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = []
for c in range(1, 6):
    f = os.path.join(REPO, "profiles", f"bench_cfg{c}_{R}.json")
    if not os.path.exists(f):
        continue
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    cfg, rf, lr, cb = d.get("results", d["config"]), d["roofline"], d.get("loop_roofline", {}), d.get("cpu_baseline", {})
    cpu = cb.get("value")
    rows.append(
        f"| {c} | {d['value']:,.1f} ({d['e2e']['value']:,.1f}) | {cfg['iterations_per_solve']} | "
        f"{d['ms_per_step'] / 1e3:.3f} s | {cfg['setup_s']:.1f} s | {cfg['time_to_solution_s']:.1f} s | "
        f"{cfg['local_operator']}, {rf['frac']:.2f} | {lr.get('frac', float('nan')):.2f} | "
        f"{cfg['device_bytes'] / 1e9:.1f} GB | {cpu:.3g} | {d['value'] / cpu:,.0f}x | {d['clocks']['sm_mhz']:.0f} |"
        if cpu else "")
print("| cfg | GPU it/s (e2e) | its | solve | setup | time-to-solution | local op., band-kernel frac "
      "| loop frac | device mem | CPU it/s | GPU/CPU | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
print("\n".join(r for r in rows if r))
