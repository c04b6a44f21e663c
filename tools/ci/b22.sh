#!/bin/bash
# 22B TP4 bench: current library, then (A/B) $OLD_LIB
i=0
for lib in lib ${OLD_LIB}; do
  i=$((i+1))
  GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so GPTB200_TIMEOUT_S=200 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29750+i)) bench.py --gpus 4 --workload gpt-22b-tp4 --no-cpu-baseline --steps ${STEPS:-5} --warmup 3 > gpurun_out/b22_$i.log 2>&1
  echo "$lib rc $?: $(tail -1 gpurun_out/b22_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), round(d["value"]), d["ms_per_step"], d["config"]["parallelism"], d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"],1) for k,v in d["kernels"].items()})' 2>&1 | tail -1)"
done
