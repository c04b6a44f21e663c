#!/bin/bash
# attention forward A/B on one GPU: parity of the two-query-tile kernel, then timing per variant
GPTB200_ATTN_FWD_2Q=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k flash 2>&1 | tail -3
for sh in "32 2048 16 128" "8 2048 16 128" "1 2048 12 128" "4 2048 16 64"; do
  timeout 120 python tools/run_attn_shape.py $sh fwd 20
  GPTB200_ATTN_FWD_PER_BLOCK=1 timeout 120 python tools/run_attn_shape.py $sh fwd 20 | sed 's/$/  (per-block 1q)/'
  GPTB200_ATTN_FWD_2Q=1 timeout 120 python tools/run_attn_shape.py $sh fwd 20 | sed 's/$/  (2q)/'
done
