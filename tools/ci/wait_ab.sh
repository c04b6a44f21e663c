#!/bin/bash
# spinning vs suspend-hinted mbarrier waits (lib_exp = -DGPTB200_WAIT_SLEEP): kernels, then the step
EXP=$PWD/paper_2312_12705_b200/lib_exp/libtrainplan_b200.so
for sh in "32 2048 16 128" "8 2048 16 128" "1 2048 12 128" "1 2048 40 160"; do
  timeout 120 python tools/run_attn_shape.py $sh fwd 20
  GPTB200_LIB=$EXP timeout 120 python tools/run_attn_shape.py $sh fwd 20 | sed 's/$/  (sleep waits)/'
  GPTB200_ATTN_FWD_2Q=1 timeout 120 python tools/run_attn_shape.py $sh fwd 20 | sed 's/$/  (2q)/'
  GPTB200_ATTN_BWD_PER_BLOCK=1 timeout 120 python tools/run_attn_shape.py $sh bwd 20 | sed 's/$/  (per-block)/'
  timeout 120 python tools/run_attn_shape.py $sh bwd 20
  GPTB200_LIB=$EXP timeout 120 python tools/run_attn_shape.py $sh bwd 20 | sed 's/$/  (sleep waits)/'
done
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/s7_bench_spin.json 2> gpurun_out/s7_bench_spin.err
GPTB200_LIB=$EXP timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/s7_bench_sleep.json 2> gpurun_out/s7_bench_sleep.err
GPTB200_ATTN_FWD_2Q=1 timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/s7_bench_spin_2q.json 2> gpurun_out/s7_bench_spin_2q.err
python - <<'PY'
import json
for f in ["spin", "sleep", "spin_2q"]:
    try:
        d = json.loads(open(f"gpurun_out/s7_bench_{f}.json").read().strip().splitlines()[-1])
        k = d.get("kernels", {})
        print(f, round(d["model_tflops_per_gpu"], 1), round(d["ms_per_step"], 1), d["clocks"]["sm_mhz"],
              {n: round(v["ms_per_step"], 2) for n, v in k.items() if v.get("ms_per_step")})
    except Exception as e:
        print(f, "failed", e)
PY
