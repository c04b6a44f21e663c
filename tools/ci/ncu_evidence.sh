#!/bin/bash
# ncu --set full evidence for the kernel families the round-1 verdict listed (1 GPU; each target runs
# once without ncu first, in the same call, then one capture).
mkdir -p gpurun_out
cap() {  # name regex count cmd...
  local name=$1 rx=$2 cnt=$3; shift 3
  "$@" > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -c $cnt \
    -o gpurun_out/ev_$name "$@" > gpurun_out/ev_$name.log 2>&1; echo "$name rc $?"
}
cap attn_fwd_hd128 fa_fwd 1 python tools/run_attn_shape.py 8 2048 16 128 fwd 1
cap ln_mbs32 "resid_ln|ln_bwd_stream" 2 python tools/run_norm_shape.py 65536 2048 0.1 1
cap gemm_22b_tp4_qkv gemm_sm100 1 python tools/run_gemm_shape.py 2048 4608 6144 0 0 0 1
cap gemm_175b_tp4_fc1 gemm_sm100 1 python tools/run_gemm_shape.py 2048 12288 12288 0 0 0 1
cap gemm_1t_tp4_fc2_dgrad gemm_sm100 1 python tools/run_gemm_shape.py 2048 25600 6400 0 1 0 1
cap gemm_1p4b_fc1_wgrad gemm_sm100 1 python tools/run_gemm_shape.py 8192 2048 65536 1 1 2 1
