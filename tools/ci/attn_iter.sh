#!/bin/bash
# Attention iteration: parity on the bounded-wait debug build (a stuck barrier traps instead of
# hanging), then the release build: parity, microbenchmark (split vs single-pass backward).
mkdir -p gpurun_out
GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_debug/libtrainplan_b200.so timeout 180 \
  python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k flash > gpurun_out/ai_dbg.log 2>&1
rc=$?; echo "debug-build parity rc $rc"; tail -3 gpurun_out/ai_dbg.log; grep -m3 HANG gpurun_out/ai_dbg.log
[ $rc -eq 0 ] || { grep -E "^E " gpurun_out/ai_dbg.log | head -20; exit 1; }
timeout 180 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k flash > gpurun_out/ai_rel.log 2>&1
rc=$?; echo "release parity rc $rc"; tail -2 gpurun_out/ai_rel.log
[ $rc -eq 0 ] || exit 1
for sh in "8 2048 16 128" "32 2048 16 128" "1 2048 12 128" "1 2048 24 128"; do
  timeout 60 python tools/run_attn_shape.py $sh bwd 10
  GPTB200_ATTN_BWD_SPLIT=0 timeout 60 python tools/run_attn_shape.py $sh bwd 10 | sed 's/$/  (single-pass)/'
done
