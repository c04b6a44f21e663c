#!/bin/bash
# attention forward variants at the tensor-parallel shapes (heads per rank): default dispatch, two-query-tile
# forced on / off, per-block grid
for shp in "1 2048 12" "1 2048 24" "2 2048 24" "4 2048 12" "1 2048 48" "2 2048 12"; do
  set -- $shp
  echo "== b=$1 s=$2 h=$3"
  python tools/run_attn_shape.py $1 $2 $3 128 fwd 20 | grep attn | sed 's/^/default  /'
  GPTB200_ATTN_FWD_2Q=1 python tools/run_attn_shape.py $1 $2 $3 128 fwd 20 | grep attn | sed 's/^/2q=1     /'
  GPTB200_ATTN_FWD_2Q=0 python tools/run_attn_shape.py $1 $2 $3 128 fwd 20 | grep attn | sed 's/^/2q=0     /'
  GPTB200_ATTN_FWD_PER_BLOCK=1 python tools/run_attn_shape.py $1 $2 $3 128 fwd 20 | grep attn | sed 's/^/perblock /'
done
