"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python scripts/launch_summary.py launches.csv [title] > profiles/rNN_launches.txt
Per kernel name: launches, total time, share of all launches, mean per launch.
The ncu pass is cold-cache and serialised: compare shares, not absolute times.
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[ui] != "ns":
            continue
        v = float(r[vi].replace(",", ""))
        name = r[ki].split("(")[0][:80]
        c = agg.setdefault(name, [0, 0.0])
        c[0] += 1
        c[1] += v
    tot = sum(v for _, v in agg.values())
    print(f"# {title}")
    print(f"# source: {path}; {sum(c for c, _ in agg.values())} launches, {tot / 1e3:.1f} us total (ncu, serialised)")
    print(f"{'launches':>8} {'total_us':>10} {'share':>6} {'mean_us':>9}  kernel")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {v / 1e3:10.1f} {v / tot * 100:5.1f}% {v / c / 1e3:9.2f}  {k}")


if __name__ == "__main__":
    main()
