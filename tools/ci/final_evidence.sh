#!/bin/bash
# Round-end evidence on one GPU for the committed build: bench line, the ncu launch list of the same
# command (per-launch gpu__time_duration, cold-cache and serialised), and ncu --set full of the step's
# top kernels at the 1.4B MBS-32 shapes (each target runs once without ncu first).
mkdir -p gpurun_out
tag=${TAG:-r02f}
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/${tag}_ncu_launches.log 2>&1; echo "launch list rc $?"
cap() {  # name regex count cmd...
  local name=$1 rx=$2 cnt=$3; shift 3
  "$@" > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -c $cnt \
    -o gpurun_out/${tag}_$name "$@" > gpurun_out/${tag}_$name.log 2>&1; echo "$name rc $?"
}
cap attn_fwd2_mbs32 fa_fwd2 1 python tools/run_attn_shape.py 32 2048 16 128 fwd 1
cap attn_bwd_mbs32 "fa_bwd_tc2|attn_dq" 2 python tools/run_attn_shape.py 32 2048 16 128 bwd 1
cap ln_mbs32 "resid_ln|ln_bwd_stream" 2 python tools/run_norm_shape.py 65536 2048 0.1 1
cap gemm_fc1_dgrad_mbs32 gemm_sm100 1 python tools/run_gemm_shape.py 65536 2048 8192 0 1 0 1
