#!/bin/bash
# Weight-gradient GEMM raster group: DRAM bytes read and duration of one launch per group size (ncu,
# single pass), for the 1.4B MBS-32 wgrad shapes (fc1: 8192x2048, fc2: 2048x8192, qkv: 6144x2048; K 65536)
for shp in "8192 2048 65536" "2048 8192 65536" "6144 2048 65536" "2048 2048 65536"; do
  set -- $shp
  for g in 0 1 2 4 8 16 32; do
    r=$(GPTB200_GEMM_GROUP=$g timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_sm100 -s 1 -c 1 --csv \
        python tools/run_gemm_shape.py $1 $2 $3 1 1 2 2 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' '{print $(NF-1)"="$NF}' | tr -d '"' | tr '\n' ' ')
    echo "M=$1 N=$2 K=$3 group=$g: $r"
  done
done
