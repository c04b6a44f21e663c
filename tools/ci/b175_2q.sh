#!/bin/bash
# 175B-shape TP4 slice: two-query-tile attention forward (new dispatch) vs forced one-tile (previous)
mkdir -p gpurun_out
i=0
for q in auto 0 auto 0; do
  i=$((i+1))
  if [ $q = auto ]; then unset GPTB200_ATTN_FWD_2Q; else export GPTB200_ATTN_FWD_2Q=0; fi
  GPTB200_TIMEOUT_S=200 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29850+i)) bench.py --gpus 4 --workload gpt-175b-slice-tp4 --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/b175q_${i}_$q.log 2>&1
  echo "2q=$q rc $?: $(tail -1 gpurun_out/b175q_${i}_$q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), d["ms_per_step"], d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"],1) for k,v in d["kernels"].items() if v["ms_per_step"]})' 2>&1 | tail -1)"
done
