"""Print the headline metrics and stall breakdown of an ncu report (first kernel).
usage: python tools/ncu_summary.py REPORT.ncu-rep [KERNEL_REGEX]"""
import csv
import io
import subprocess
import sys

cmd = ["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"]
if len(sys.argv) > 2:
    cmd += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:55s} {v[i]} {units[i]}")
items = []
for i, x in enumerate(h):
    if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("not_issued"):
        try:
            items.append((float(v[i].replace(",", "")), x))
        except ValueError:
            pass
items.sort(reverse=True)
tot = sum(a for a, _ in items) or 1
print("stalls:", ", ".join(f"{b.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * a / tot:.1f}%"
                           for a, b in items[:8]))
