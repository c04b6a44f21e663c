#!/bin/bash
for sh in "8 2048 16 128" "32 2048 16 128"; do
  timeout 60 python tools/run_attn_shape.py $sh bwd 10
  GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_exp/libtrainplan_b200.so timeout 60 python tools/run_attn_shape.py $sh bwd 10 | sed 's/$/  (no dQ flush)/'
done
