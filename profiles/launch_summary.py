"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file`)
into per-kernel launches / total time / share, libtgs kernels first, then torch's own.

    python profiles/launch_summary.py <launches.csv> "<command line>" > <summary.txt>

Launches under ncu are serialised and cold-cache: compare SHARES, not absolute times.
"""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)  # drop the parameter list
    return name.replace("void ", "").strip()


def main(path: str, cmd: str) -> None:
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r["Metric Unit"], 1.0)
        rows.append((short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")) * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for k, us in rows:
        agg[k][0] += 1
        agg[k][1] += us
    total = sum(v[1] for v in agg.values())
    ours = {k: v for k, v in agg.items() if k.startswith("tgs::")}
    other = {k: v for k, v in agg.items() if not k.startswith("tgs::")}
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none\n    {cmd}")
    print(f"{len(rows)} launches ({sum(v[0] for v in ours.values())} libtgs), cold-cache and serialised: "
          "compare SHARES, not absolute times")
    print(f"{'kernel':58s} {'launches':>8s} {'us total':>10s} {'us/launch':>10s} {'share':>7s}")
    for group in (ours, other):
        for k, (n, us) in sorted(group.items(), key=lambda kv: -kv[1][1]):
            print(f"{k[:58]:58s} {n:8d} {us:10.1f} {us / n:10.1f} {100 * us / total:6.1f}%")
        print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
