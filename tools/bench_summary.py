"""Compact one-line summary of bench.py JSON lines read from stdin (debug helper)."""
import json
import sys

for line in sys.stdin:
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    ks = {k: round(v["ms_per_step"], 1) for k, v in d.get("kernels", {}).items()}
    print(d["config"].get("parallelism"), f"tok/s {d['value']:.0f}", f"TF/GPU {d.get('model_tflops_per_gpu', 0):.1f}",
          f"ms {d['ms_per_step']:.1f}", f"clk {d.get('clocks', {}).get('sm_mhz')}", ks, flush=True)
