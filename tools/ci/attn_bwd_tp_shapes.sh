#!/bin/bash
# attention backward variants at the tensor-parallel per-rank shapes (hd 128): default dispatch vs
# per-block grid forced on / off
for shp in "1 2048 12" "1 2048 24" "2 2048 24" "4 2048 12" "1 2048 48" "8 2048 16"; do
  set -- $shp
  echo "== b=$1 s=$2 h=$3"
  python tools/run_attn_shape.py $1 $2 $3 128 bwd 20 | grep attn | sed 's/^/default  /'
  GPTB200_ATTN_BWD_PER_BLOCK=1 python tools/run_attn_shape.py $1 $2 $3 128 bwd 20 | grep attn | sed 's/^/perblock /'
  GPTB200_ATTN_BWD_PER_BLOCK=0 python tools/run_attn_shape.py $1 $2 $3 128 bwd 20 | grep attn | sed 's/^/persist  /'
done
