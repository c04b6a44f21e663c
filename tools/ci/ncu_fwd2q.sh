#!/bin/bash
export GPTB200_ATTN_FWD_2Q=1
python tools/run_attn_shape.py 8 2048 16 128 fwd 3 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:fa_fwd2 -c 1 -o gpurun_out/ncu_fwd2q python tools/run_attn_shape.py 8 2048 16 128 fwd 1 > gpurun_out/ncu_fwd2q.log 2>&1; echo rc $?
