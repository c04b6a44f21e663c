#!/bin/bash
# 1-GPU check of the tree: GPU tests, then the headline bench (default) and an A/B bench
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/c_pytest.log
tail -3 gpurun_out/c_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
eval "$AB_ENV timeout 300 python bench.py --steps 10 --warmup 3" > gpurun_out/c_bench_ab.json 2> gpurun_out/c_bench_ab.err
python - <<'PY'
import json
for f in ["c_bench", "c_bench_ab"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        k = d.get("kernels", {})
        print(f, round(d["model_tflops_per_gpu"], 1), round(d["ms_per_step"], 1), d["clocks"]["sm_mhz"], d["e2e"]["value"],
              {n: (round(v["ms_per_step"], 2), round(v.get("tflops", v.get("gbs", 0)) or 0)) for n, v in k.items() if v.get("ms_per_step")})
    except Exception as e:
        print(f, "failed", e)
PY
