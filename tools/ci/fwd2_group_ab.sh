#!/bin/bash
# L2-grouped launch order of the two-query-tile attention forward (lib) vs heaviest-first over all heads
# (lib_old): DRAM bytes of one launch at the 1.4B MBS-32 shape, then the 1.4B bench alternating
mkdir -p gpurun_out
for lib in lib lib_old; do
  GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so python tools/run_attn_shape.py 32 2048 16 128 fwd 2 > /dev/null 2>&1
  GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum \
    --clock-control none -k regex:fa_fwd2 -c 1 --csv python tools/run_attn_shape.py 32 2048 16 128 fwd 2 2>/dev/null | grep -E "dram__bytes|duration" | sed "s/^/$lib /"
done
LIBS="lib lib_old lib lib_old lib lib_old" bash tools/ci/lib_ab.sh
