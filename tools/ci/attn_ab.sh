#!/bin/bash
# attention backward A/B on one GPU: parity (default / forced per-block) then timing per variant
set -x
python -m pytest tests/test_gpu_kernels.py -q -x -k flash 2>&1 | tail -3
GPTB200_ATTN_BWD_PER_BLOCK=1 python -m pytest tests/test_gpu_kernels.py -q -x -k flash 2>&1 | tail -3
for sh in "32 2048 16 128" "8 2048 16 128"; do
  GPTB200_ATTN_BWD_PER_BLOCK=1 timeout 120 python tools/run_attn_shape.py $sh bwd 20
  GPTB200_ATTN_BWD_PER_BLOCK=1 GPTB200_ATTN_BWD_SMEM_P=1 timeout 120 python tools/run_attn_shape.py $sh bwd 20 | sed 's/$/  (P in smem)/'
done
