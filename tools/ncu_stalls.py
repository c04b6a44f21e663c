"""Summarise an ncu report: key throughput metrics + top stall PCs + mbarrier waits by name
(debug helper; usage: python tools/ncu_stalls.py report.ncu-rep [kernel-regex])."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_op_red.sum", "launch__registers_per_thread"]
for k in want:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                      text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hh, data = rows[1], rows[2:]
i_s = hh.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[i_s]) for x in data if x[i_s].isdigit())
a0 = int(data[0][0], 16)
print("samples", tot)
for x in sorted(data, key=lambda x: -int(x[i_s]) if x[i_s].isdigit() else 0)[:25]:
    print(f"{int(x[0], 16) - a0:6x} {int(x[i_s]):6d} {100 * int(x[i_s]) / tot:5.1f}%  {x[1][:90]}")
print("mbarrier waits (try-wait + retry branch samples) by smem offset:")
agg = {}
for k, x in enumerate(data):
    if "TRYWAIT" in x[1]:
        m = re.search(r"\+0x([0-9a-f]+)\]", x[1])
        n = (int(x[i_s]) if x[i_s].isdigit() else 0) + (int(data[k + 1][i_s]) if data[k + 1][i_s].isdigit() else 0)
        agg[m.group(1) if m else "?"] = agg.get(m.group(1) if m else "?", 0) + n
for k2, n in sorted(agg.items(), key=lambda t: -t[1]):
    print(f"  +0x{k2}: {n} ({100 * n / tot:.1f}%)")
