"""Per-instruction stall breakdown of one kernel in an ncu report (source page, SASS):
python tools/ncu_source_stalls.py report.ncu-rep [top]  -> totals per stall reason, top instructions."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
lines = txt.splitlines()
# first block only (one kernel): header line 2, rows until the next "Kernel Name" line
start = 1
end = next((i for i in range(2, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
h = rows[0]
data = rows[1:]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {r: 0 for r in reasons}
samples = h.index("Warp Stall Sampling (All Samples)")
allsum = 0
for x in data:
    for r in reasons:
        v = x[h.index(r)]
        tot[r] += int(v) if v.isdigit() else 0
    allsum += int(x[samples]) if x[samples].isdigit() else 0
print(f"samples {allsum}")
for r, v in sorted(tot.items(), key=lambda t: -t[1])[:12]:
    print(f"  {r:28s} {v:8d} {100 * v / max(allsum, 1):5.1f}%")
a0 = int(data[0][0], 16)
print("top instructions:")
for x in sorted(data, key=lambda x: -(int(x[samples]) if x[samples].isdigit() else 0))[:top]:
    s = int(x[samples]) if x[samples].isdigit() else 0
    dom = max(reasons, key=lambda r: int(x[h.index(r)]) if x[h.index(r)].isdigit() else 0)
    print(f"  {int(x[0], 16) - a0:6x} {s:6d} {100 * s / max(allsum, 1):5.1f}% {dom[6:]:14s} {x[1].strip()[:80]}")
