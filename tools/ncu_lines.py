#!/usr/bin/env python3
"""Summarise an ncu report's source page by CUDA source line.

usage: tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]
Prints the source lines with the most warp-stall samples, plus shared-memory
bank-conflict wavefronts and L2 sector excess per line.
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, recs = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {k: i for i, k in enumerate(r) if k not in ("Source",)}
            continue
        if hdr and r[0].isdigit() and len(r) > 4 and r[2] == "-":
            def g(name):
                i = hdr.get(name)
                try:
                    return float(r[i]) if i is not None else 0.0
                except ValueError:
                    return 0.0
            recs.append((g("Warp Stall Sampling (All Samples)"), fname, int(r[0]), r[1][:90],
                         g("L1 Wavefronts Shared Excessive"), g("L2 Theoretical Sectors Global Excessive"),
                         g("Instructions Executed")))
    tot = sum(x[0] for x in recs) or 1
    for s, f, ln, src, bank, l2x, ins in sorted(recs, key=lambda x: -x[0])[:top]:
        print(f"{100*s/tot:5.1f}% {f}:{ln:<5} inst={ins:>10.0f} bankX={bank:>9.0f} l2X={l2x:>9.0f}  {src}")


if __name__ == "__main__":
    main()
