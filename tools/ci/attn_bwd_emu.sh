#!/bin/bash
for emu in 1 2; do GPTB200_ATTN_BWD_EMU=$emu GPTB200_ATTN_BWD_PER_BLOCK=1 timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -k flash 2>&1 | tail -1; done
for sh in "32 2048 16 128" "8 2048 16 128"; do
  for emu in 0 1 2 3; do
    GPTB200_ATTN_BWD_EMU=$emu timeout 120 python tools/run_attn_shape.py $sh bwd 20 | sed "s/\$/  (emu $emu)/"
  done
done
