#!/bin/bash
# attention fwd/bwd at the TP-rank-local shapes of the BASELINE layouts, persistent vs per-block
for shape in "1 2048 12 128" "1 2048 6 128" "1 2048 24 128" "1 2048 40 160" "1 2048 20 160" "32 2048 16 128"; do
  timeout 120 python tools/run_attn_shape.py $shape fwd 10
  GPTB200_ATTN_FWD_PER_BLOCK=1 timeout 120 python tools/run_attn_shape.py $shape fwd 10 | sed 's/$/  (per-block)/'
  timeout 120 python tools/run_attn_shape.py $shape bwd 10
done
