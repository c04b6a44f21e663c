#!/bin/bash
# sustained GEMMs at the MBS-32 step shapes, lib vs lib_old, twice each (same box)
for lib in lib lib_old lib lib_old; do
  echo "== $lib"; GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so SHAPES=${SHAPES:-mbs32} timeout 400 python tools/bench_gemm_sustained.py 2>&1 | grep "^ours"
done
