#!/bin/bash
# Attention iteration: parity on the bounded-wait debug build (a stuck barrier traps instead of
# hanging), then the release build: parity, microbenchmark, backward timeline trace.
mkdir -p gpurun_out
GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_debug/libtrainplan_b200.so timeout 180 \
  python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k flash > gpurun_out/ai_dbg.log 2>&1
rc=$?; echo "debug-build parity rc $rc"; tail -3 gpurun_out/ai_dbg.log; grep -m3 HANG gpurun_out/ai_dbg.log
[ $rc -eq 0 ] || exit 1
timeout 180 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k flash > gpurun_out/ai_rel.log 2>&1
rc=$?; echo "release parity rc $rc"; tail -2 gpurun_out/ai_rel.log
[ $rc -eq 0 ] || exit 1
timeout 300 python tools/bench_attn.py bwd 2>&1 | tee gpurun_out/ai_bench.log
GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_trace/libtrainplan_b200.so GPTB200_ATTN_TRACE=gpurun_out/trace128.csv \
  timeout 120 python tools/run_attn_shape.py 8 2048 16 128 bwd 2 > /dev/null && python tools/attn_trace.py gpurun_out/trace128.csv | tail -9
