"""Top SASS lines of one kernel in an ncu report by stall samples.
usage: python tools/ncu_hotsass.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
r = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = r[0]
si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
rows = [x for x in r[1:] if len(x) == len(h) and x[0].startswith("0x")]
tot = sum(float(x[si] or 0) for x in rows) or 1
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
for x in sorted(rows, key=lambda x: -float(x[si] or 0))[:n]:
    print(f"{100 * float(x[si] or 0) / tot:5.1f}%  {x[ii]:>12}  {x[1].strip()[:90]}")
