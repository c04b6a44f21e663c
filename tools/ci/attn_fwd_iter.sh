#!/bin/bash
mkdir -p gpurun_out
GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_debug/libtrainplan_b200.so timeout 180 \
  python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k flash > gpurun_out/af_dbg.log 2>&1
rc=$?; echo "debug-build parity rc $rc"; tail -2 gpurun_out/af_dbg.log; [ $rc -eq 0 ] || { grep -E "^E " gpurun_out/af_dbg.log | head; exit 1; }
timeout 180 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k flash > gpurun_out/af_rel.log 2>&1
rc=$?; echo "release parity rc $rc"; tail -2 gpurun_out/af_rel.log; [ $rc -eq 0 ] || exit 1
for sh in "32 2048 16 128" "8 2048 16 128" "1 2048 12 128" "1 2048 40 160"; do
  timeout 60 python tools/run_attn_shape.py $sh fwd 20
  GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_old/libtrainplan_b200.so timeout 60 python tools/run_attn_shape.py $sh fwd 20 | sed 's/$/  (previous)/'
done
