"""Per-CUDA-source-line stall samples of one kernel in an ncu report.
usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, agg, hdr = "", {}, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].isdigit():
        s = float(r[4] or 0)
        key = (fname, int(r[0]))
        a = agg.setdefault(key, [0.0, 0, r[1]])
        a[0] += s
        a[1] += int(float(r[7] or 0))
tot = sum(v[0] for v in agg.values()) or 1
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
for (f, ln), (s, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * s / tot:5.1f}% {ex:>12} {f}:{ln:<5} {src.strip()[:90]}")
