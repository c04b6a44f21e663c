#!/bin/bash
for sh in "8 2048 16 128"; do
  GPTB200_ATTN_FWD_2Q=1 timeout 120 python tools/run_attn_shape.py $sh fwd 5 | sed 's/$/  (2q)/'
  GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_debug/libtrainplan_b200.so GPTB200_ATTN_FWD_2Q=1 timeout 120 python tools/run_attn_shape.py $sh fwd 5 | sed 's/$/  (2q, spin waits)/'
done
