#!/bin/bash
# Attention kernels: parity tests, microbenchmark, then (if both passed) one ncu capture per backward variant.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "flash" > gpurun_out/attn_tests.log 2>&1
rc=$?; echo "pytest rc $rc" >> gpurun_out/attn_tests.log; tail -5 gpurun_out/attn_tests.log
[ $rc -eq 0 ] || exit 1
timeout 300 python tools/bench_attn.py > gpurun_out/attn_bench.log 2>&1; echo "bench rc $?"; cat gpurun_out/attn_bench.log
if [ -n "${NCU:-}" ]; then
  python tools/run_attn_shape.py 1 2048 40 160 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_ -c 4 -o gpurun_out/${NCU} \
     python tools/run_attn_shape.py 1 2048 40 160 > gpurun_out/${NCU}.log 2>&1; echo "ncu rc $?"
fi
