#!/bin/bash
GPTB200_ATTN_FWD_2Q=1 timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -k flash 2>&1 | tail -2
for cs in 2; do for emu in 0 2 3; do
  for sh in "32 2048 16 128" "8 2048 16 128"; do
    GPTB200_ATTN_FWD_CS=$cs GPTB200_ATTN_FWD_EMU=$emu GPTB200_ATTN_FWD_2Q=1 timeout 120 python tools/run_attn_shape.py $sh fwd 20 | sed "s/\$/  (2q cs $cs emu $emu)/"
  done
done; done
GPTB200_ATTN_FWD_2Q=1 GPTB200_LIB=$PWD/paper_2312_12705_b200/lib_trace/libtrainplan_b200.so GPTB200_ATTN_TRACE=gpurun_out/trace_fwd.csv \
  timeout 120 python tools/run_attn_shape.py 8 2048 16 128 fwd 1; echo "rc $?"
python tools/attn_fwd_trace.py gpurun_out/trace_fwd.csv
