"""Timeline of one backward CTA from a GPTB200_ATTN_TRACE dump (debug build, lib_trace):
python tools/attn_trace.py trace.csv  -> per query tile, cycles relative to the first S issue."""
import sys

import numpy as np

t = np.loadtxt(sys.argv[1], delimiter=",", dtype=np.float64)
n = int((t[:, 2] > 0).sum())
t = t[:n]
base = t[0, 2]
names = {0: "mma:wait_q", 1: "mma:st_free", 2: "mma:S_issued", 3: "st2:start", 4: "st2:pds_ok", 5: "st2:dq_free",
         6: "st2:issued", 9: "cmp:s_ready", 10: "cmp:ldtm", 11: "cmp:math_done", 12: "cmp:pds_free", 13: "cmp:pds_full",
         14: "fl:dq_ready", 15: "fl:done", 16: "cmp:st_smem", 17: "cmp:fence", 18: "cmp:st_tmem"}
print("tile " + " ".join(f"{v:>13s}" for v in names.values()))
for j in range(n):
    print(f"{j:4d} " + " ".join(f"{(t[j, k] - base) if t[j, k] else float('nan'):13.0f}" for k in names))
d = np.diff(t[:, 2])
print(f"S issue period: median {np.median(d):.0f} cycles/tile  (tensor floor 1280 for hd 128, 64-q tiles)")
for a, b, lab in [(9, 10, "s_ready -> ldtm done"), (10, 11, "math"), (11, 13, "pds_free wait + store + fence"),
                  (2, 9, "S issued -> compute sees S"), (13, 4, "pds_full -> stage 2 sees it"),
                  (14, 15, "dq flush"), (12, 16, "smem stores"), (16, 17, "fence.proxy.async"),
                  (17, 18, "tcgen05.wait::st"), (18, 13, "tc fence + arrive"), (6, 14, "stage2 issued -> dq ready")]:
    v = t[:, b] - t[:, a]
    v = v[(t[:, a] > 0) & (t[:, b] > 0)]
    if len(v):
        print(f"{lab:32s} median {np.median(v):8.0f}  p90 {np.percentile(v, 90):8.0f}")
