#!/bin/bash
GPTB200_ATTN_BWD_Q128=1 timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -k flash 2>&1 | tail -2
for sh in "32 2048 16 128" "8 2048 16 128" "1 2048 12 128"; do
  timeout 120 python tools/run_attn_shape.py $sh bwd 20
  GPTB200_ATTN_BWD_Q128=1 timeout 120 python tools/run_attn_shape.py $sh bwd 20 | sed 's/$/  (q128)/'
done
