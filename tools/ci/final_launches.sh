#!/bin/bash
# ncu launch list of the last build's bench command and one ncu --set full of the fc1 weight-gradient GEMM
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02z_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/r02z_ncu_launches.log 2>&1; echo "launch list rc $?"
python tools/run_gemm_shape.py 8192 2048 65536 1 1 2 2 > /dev/null 2>&1 && timeout 300 ncu --set full --clock-control none --import-source on \
  -k regex:gemm_sm100 -s 1 -c 1 -o gpurun_out/r02z_gemm_fc1_wgrad python tools/run_gemm_shape.py 8192 2048 65536 1 1 2 2 > gpurun_out/r02z_wgrad.log 2>&1; echo "wgrad rc $?"
