#!/bin/bash
mkdir -p gpurun_out
GPTB200_ATTN_BWD_PER_BLOCK=1 GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_trace/libtrainplan_b200.so GPTB200_ATTN_TRACE=gpurun_out/trace128.csv \
  timeout 120 python tools/run_attn_shape.py 8 2048 16 128 bwd 2; echo "rc $?"
python tools/attn_trace.py gpurun_out/trace128.csv
