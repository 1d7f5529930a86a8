#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list.

usage: tools/launch_summary.py launches.csv [title]
Per kernel: launches, mean duration (us) and share of the per-step kernels
(kernels launched once per timed step; one-off setup launches are listed
separately).  ncu serialises launches with cold caches, so compare SHARES
with bench.py's live per-kernel times, not absolute durations.
"""
import collections
import csv
import io
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    ix = {h: i for i, h in enumerate(rows[0])}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) < len(ix) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").strip()
        agg.setdefault(name, []).append(float(r[ix["Metric Value"]]) * SCALE[r[ix["Metric Unit"]]])
    steps = max(len(v) for v in agg.values())
    per_step = {k: v for k, v in agg.items() if len(v) == steps}
    other = {k: v for k, v in agg.items() if len(v) != steps}
    tot = sum(sum(v) for v in per_step.values())
    print(f"# {title}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised launches")
    print(f"# per-step kernels (launched {steps}x)")
    print("kernel,launches,mean_us,share")
    for k, v in sorted(per_step.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k},{len(v)},{sum(v) / len(v):.2f},{sum(v) / tot:.3f}")
    print(f"# per-step total (sum of means): {tot / steps:.2f} us")
    if other:
        print("# setup / one-off launches (outside the timed step)")
        for k, v in other.items():
            print(f"{k},{len(v)},{sum(v) / len(v):.2f},-")


if __name__ == "__main__":
    main()
