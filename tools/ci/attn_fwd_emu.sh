#!/bin/bash
GPTB200_ATTN_FWD_2Q=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k flash 2>&1 | tail -2
for emu in 0 1 2 3 4; do
  for sh in "32 2048 16 128" "8 2048 16 128"; do
    GPTB200_ATTN_FWD_EMU=$emu GPTB200_ATTN_FWD_2Q=1 timeout 120 python tools/run_attn_shape.py $sh fwd 20 | sed "s/\$/  (2q emu $emu)/"
  done
done
