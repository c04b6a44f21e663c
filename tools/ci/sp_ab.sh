#!/bin/bash
# SP LayerNorm kernels in isolation on 4 GPUs: previous build (lib_old) vs current
for lib in lib_old lib; do
  for d in "6144 48" "12288 96" "25600 160"; do
    set -- $d
    GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so timeout 300 python -m torch.distributed.run \
      --nnodes=1 --nproc-per-node ${NP:-4} --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) \
      tools/bench_sp.py --hidden $1 --heads $2 2>&1 | grep -E "sp_ln|nvls" | sed "s/^/$lib /"
  done
done
