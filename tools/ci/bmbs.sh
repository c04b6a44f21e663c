#!/bin/bash
# TP workloads at larger micro-batches on one 4-GPU box (WORKLOADS="..." overrides the list)
mkdir -p gpurun_out
i=0
for w in ${WORKLOADS:-gpt-22b-tp4-mbs8 gpt-175b-slice-tp4-mbs2 gpt-175b-slice-tp4-mbs4 gpt-175b-slice-tp2pp2-mbs2}; do
  i=$((i+1))
  GPTB200_TIMEOUT_S=200 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29770+i)) bench.py --gpus 4 --workload $w --no-cpu-baseline --steps ${STEPS:-3} --warmup 2 $EXTRA > gpurun_out/bmbs_$w.log 2>&1
  echo "$w rc $?: $(tail -1 gpurun_out/bmbs_$w.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), round(d["value"]), d["ms_per_step"], d["config"]["parallelism"], d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"],1) for k,v in d["kernels"].items()})' 2>&1 | tail -1)"
done
