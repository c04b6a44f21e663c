#!/bin/bash
# ncu --set full of the fc1 forward GEMM with the bias+GeLU dual-output epilogue vs the plain epilogue (1.4B MBS-32 shape)
mkdir -p gpurun_out
cap() {
  local name=$1; shift
  "$@" > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -c 1 \
    -o gpurun_out/ev_$name "$@" > gpurun_out/ev_$name.log 2>&1; echo "$name rc $?"
}
cap fc1_gelu python tools/run_gemm_shape.py 65536 8192 2048 0 0 1 1
cap fc1_plain python tools/run_gemm_shape.py 65536 8192 2048 0 0 0 1
