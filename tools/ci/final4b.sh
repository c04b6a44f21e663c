#!/bin/bash
# 22B TP4 and DP4 bench lines on the final build (4 GPUs)
mkdir -p gpurun_out
i=0
for w in "gpt-22b-tp4" "gpt-1.4b" "gpt-22b-tp4"; do
  i=$((i+1))
  GPTB200_TIMEOUT_S=200 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29960+i)) bench.py --gpus 4 --workload $w --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/f4c_${i}_$w.json 2> gpurun_out/f4c_${i}_$w.err
  echo "$w rc $?: $(tail -1 gpurun_out/f4c_${i}_$w.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), round(d["value"]), d["ms_per_step"], d["config"]["parallelism"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
done
