"""Hottest SASS windows of an ncu report (instructions executed, stall samples).
usage: python tools/ncu_hot.py REPORT.ncu-rep [window] [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 16
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
ia, isrc, ist = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
num = lambda x: float(x or 0)
tot = sum(num(r[ia]) for r in data) or 1
tst = sum(num(r[ist]) for r in data) or 1
print(f"total {tot:.3e} inst, {tst:.0f} samples")
win = []
for i in range(0, len(data), W):
    ch = data[i:i + W]
    win.append((sum(num(r[ia]) for r in ch), sum(num(r[ist]) for r in ch), i))
for a, b, i in sorted(win, reverse=True)[:top]:
    ops = " ".join(r[isrc].split()[0] if not r[isrc].strip().startswith("@") else r[isrc].split()[1]
                   for r in data[i:i + W] if r[isrc].strip())
    print(f"{100 * a / tot:5.1f}% inst {100 * b / tst:5.1f}% stall @{i}: {ops[:150]}")
