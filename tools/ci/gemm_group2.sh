#!/bin/bash
# Forward / dgrad GEMM raster group at the 1.4B MBS-32 shapes: DRAM bytes + duration per group (ncu single pass)
for shp in "65536 6144 2048 0 0 0" "65536 8192 2048 0 0 1" "65536 2048 2048 0 0 0" "65536 2048 8192 0 0 0" "65536 2048 8192 0 1 0" "65536 2048 6144 0 1 0" "65536 2048 2048 0 1 0"; do
  set -- $shp
  for g in 1 2 4 8 16 32; do
    r=$(GPTB200_GEMM_GROUP=$g timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_sm100 -s 1 -c 1 --csv \
        python tools/run_gemm_shape.py $1 $2 $3 $4 $5 $6 2 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' '{print $(NF-1)"="$NF}' | tr -d '"' | tr '\n' ' ')
    echo "M=$1 N=$2 K=$3 mn=$4$5 epi=$6 group=$g: $r"
  done
done
