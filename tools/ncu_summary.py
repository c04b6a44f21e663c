"""Summarise an ncu report (one line per captured launch) or an ncu launch-list CSV (per-kernel
shares): python tools/ncu_summary.py full <report.ncu-rep> | launches <launches.csv>."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
           "launch__registers_per_thread", "sm__inst_issued.avg.pct_of_peak_sustained_active"]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        parts = [f"Kernel Name={d.get('Kernel Name', '')}", f"Grid Size={d.get('Grid Size', '')}",
                 f"Block Size={d.get('Block Size', '')}"]
        for m in METRICS:
            if m in h:
                parts.append(f"{m}={d[m]} {units[h.index(m)]}")
        print(" | ".join(parts))


def launches(path):
    tot, cnt = defaultdict(float), defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.reader(io.StringIO("".join(lines)))
    h = next(r)
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    for row in r:
        if row[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", row[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
        name = re.sub(r"^.*::", "", name)
        tot[name] += float(row[vi].replace(",", ""))
        cnt[name] += 1
    t = sum(tot.values())
    print(f"# total {t / 1e6:.1f} ms (ns units below), {sum(cnt.values())} launches")
    print("kernel,launches,total_ns,share")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k},{cnt[k]},{v:.0f},{v / t:.4f}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
