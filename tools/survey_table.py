"""BASELINE.md §4 rows from committed bench lines (profiles/r02_survey_*.json)."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
order = ["C1", "C2_1e-4", "C2_1e-3", "C2_1e-2", "C3_1e-3", "C3_1e-4", "C3_1e-5", "C3_1e-6", "default", "C4_1e-5",
         "C4_1.2e-4_t100", "C4_1.2e-4_capped"]
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
print("| Config | ξ_rel | GPUs | N | \\|V\\| | \\|E\\| | iterations (stop) | t S1–S5 (ms) | Mp/s | Mp/s incl. check | "
      "K3 frac of HBM | K2 count tests/s | MCC after | oracle, 1 core (Mp/s; sample N) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for name in order:
    p = os.path.join(ROOT, "profiles", f"{tag}_survey_{name}.json")
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    c, r = d["config"], d["result"]
    stop = "converged" if r["converged"] else ("T_max" if d["config"]["stop"].startswith("fixed") is False else "fixed")
    if "fixed" in d["config"]["stop"]:
        stop = f"fixed {d['config']['t_max']}"
    elif not r["converged"]:
        stop = f"T_max={d['config']['t_max']}, not converged"
    k3 = (d.get("k3_roofline") or {}).get("frac")
    pt = (d.get("pair_tests") or {}).get("K2_count", {}).get("tests_per_s")
    cb = d.get("cpu_baseline") or {}
    cbs = f"{cb['value']:.3f} ({cb['sample'].split(' at N=')[1].split(' ')[0]})" if cb.get("value") else "—"
    print(f"| {c['workload']} | {c['xi_rel']:g} | {d['n_gpus']} | {c['n']:,} | {r['n_pairs']:,} | {r['n_editable']:,} | "
          f"{r['iterations']} ({stop}) | {d['ms_per_step']:.2f} | {d['value']:.1f} | {d['incl_check']['value']:.1f} | "
          f"{k3:.3f} | {pt / 1e9:.1f} G | {r['mcc_after']:.6f} | {cbs} |" if k3 is not None and pt else
          f"| {c['workload']} | {c['xi_rel']:g} | {d['n_gpus']} | {c['n']:,} | {r['n_pairs']:,} | {r['n_editable']:,} | "
          f"{r['iterations']} ({stop}) | {d['ms_per_step']:.2f} | {d['value']:.1f} | {d['incl_check']['value']:.1f} | "
          f"{k3 if k3 is not None else '—'} | {'%.1f G' % (pt / 1e9) if pt else '—'} | {r['mcc_after']:.6f} | {cbs} |")
