"""Shared-memory wavefronts per CUDA source line of one kernel in an ncu report.
usage: python tools/ncu_smem_lines.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
fname, hdr, agg = "", None, []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Name":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        f = lambda k: float((d.get(k) or "0").replace(",", "") or 0)
        if f("L1 Wavefronts Shared"):
            agg.append((f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Ideal"), f("Instructions Executed"),
                        f"{fname}:{r[0]}", r[1].strip()[:80]))
tot = sum(a[0] for a in agg) or 1
print(f"total shared wavefronts {tot:.4g}")
for w, i, ins, loc, src in sorted(agg, reverse=True)[:n]:
    print(f"{100 * w / tot:5.1f}% {w:12.4g} ideal {i:12.4g} inst {ins:11.4g} {loc:22s} {src}")
