#!/bin/bash
# hd-160 attention on the bounded-wait debug build first (a stuck barrier prints and traps), then the
# release build; short per-test timeouts.
mkdir -p gpurun_out
for lib in lib_debug lib; do
  for t in "2-256-2-160" "1-2048-4-160" "2-384-3-160"; do
    GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so GPTB200_ATTN_SYNC_DEBUG=1 timeout 90 \
      python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "flash and $t" > gpurun_out/attn_dbg_${lib}_$t.log 2>&1
    rc=$?; echo "$lib $t rc $rc"; grep -E "HANG|attention bwd|fa_bwd_tc3|passed|failed|Error|assert" gpurun_out/attn_dbg_${lib}_$t.log | head -4
    [ $rc -eq 0 ] || exit 1
  done
done
