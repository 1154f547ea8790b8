# Rows of DESIGN.md section 10 / README performance table from profiles/<tag>_bench_*.json
# usage: python scripts/bench_table.py r2g
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r2g"


def last_line(path):
    with open(path) as fh:
        lines = [l for l in fh.read().strip().splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


names = {"C0": "C0 (2D N=64 p=5)", "C1": "C1 (2D N=1024 p=7)", "C2": "C2 (2D N=16384 p=9)",
         "C3": "C3 (3D N=128 p=5)", "C4": "C4 (3D N=512 p=7)", "C2_f32": "C2 FP32 variant"}
print("| config | Mpoints/s (e2e) | step ms | apply ms | plan ms | translate ms | HBM frac | FP64 frac |")
print("|---|---|---|---|---|---|---|---|")
for c in ("C0", "C1", "C2", "C3", "C4", "C2_f32"):
    try:
        d = last_line(f"profiles/{tag}_bench_{c}.json")
    except Exception as e:  # missing leg: say so
        print(f"| {names[c]} | missing ({e.__class__.__name__}) |")
        continue
    r = d["roofline"]
    km = r["kernel_ms"]
    bw_ev = r.get("achieved_per_level_events")
    frac_ev = bw_ev / r["peak"] if bw_ev else float("nan")
    fp = r.get("fp64", {}).get("frac", float("nan"))
    print(f"| {names[c]} | {d['value']:.4g} ({d['e2e']['value']:.4g}) | {d['ms_per_step']:.4g} | "
          f"{d['apply_ms']:.4g} | {d['plan_ms']:.4g} | {km['translate_total']:.4g} "
          f"({km['translate_per_level_events']:.4g}) | {r['frac']:.3f} ({frac_ev:.3f}) | {fp:.3f} |")
    if "accuracy" in d:
        a = d["accuracy"]
        print(f"<!-- {c} accuracy: direct {a.get('rel_l2_vs_direct')}, oracle {a.get('rel_l2_vs_oracle_butterfly')} "
              f"leaf {km.get('leaf')} final {km.get('final')} clocks {d.get('clocks')} -->")
