"""Timeline of one two-query-tile forward CTA from a GPTB200_ATTN_TRACE dump (debug build, lib_trace):
python tools/attn_fwd_trace.py trace.csv -> per kv tile, cycles relative to the first stamp."""
import sys

import numpy as np

t = np.loadtxt(sys.argv[1], delimiter=",", dtype=np.float64)
n = int((t[:, 3] > 0).sum())
t = t[:n]
base = t[t > 0].min()
names = {0: "mma:p0", 1: "mma:iss0", 2: "mma:p1", 3: "mma:iss1", 4: "sm0:wait", 5: "sm0:S", 6: "sm0:max", 7: "sm0:exp",
         8: "sm0:arr", 9: "sm1:wait", 10: "sm1:S", 11: "sm1:max", 12: "sm1:exp", 13: "sm1:arr"}
print("kv  " + " ".join(f"{v:>9s}" for v in names.values()))
for j in range(n):
    print(f"{j:3d} " + " ".join(f"{(t[j, k] - base) if t[j, k] else float('nan'):9.0f}" for k in names))
for a, b, lab in [(5, 6, "sm0 S seen -> max done (ld + max)"), (6, 7, "sm0 max -> exps done"), (7, 8, "sm0 st wait + arrive"),
                  (8, 0, "sm0 arrive -> mma sees p0"), (1, 5, "mma issued PV0/S0 -> sm0 sees S0(j+1)"),
                  (10, 11, "sm1 ld + max"), (11, 12, "sm1 exps"), (3, 10, "mma issued PV1/S1 -> sm1 sees S1(j+1)")]:
    if b in (0,) or a in (1, 3):
        v = t[1:, b] - t[:-1, a] if a in (1, 3) else t[:, b] - t[:, a]
    else:
        v = t[:, b] - t[:, a]
    v = v[np.isfinite(v) & (v > 0) & (v < 1e7)]
    if len(v):
        print(f"{lab:40s} median {np.median(v):7.0f}  p90 {np.percentile(v, 90):7.0f}")
print(f"kv-tile period (mma:iss1): median {np.median(np.diff(t[:, 3])):.0f} cycles (tensor floor 2048 for hd 128)")
