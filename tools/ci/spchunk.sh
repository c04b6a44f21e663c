#!/bin/bash
# Row-chunked SP forward: multi-GPU parity with 2 (and 4) chunks forced on the SP layouts, then the
# 22B TP4 bench with 1 / 2 / 4 chunks on one 4-GPU box
mkdir -p gpurun_out
GPTB200_SP_FWD_CHUNKS=2 timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "tp2 or tp4" > gpurun_out/spc_tests2.log 2>&1; echo "tests chunks=2 rc $?"; tail -2 gpurun_out/spc_tests2.log
GPTB200_SP_FWD_CHUNKS=4 timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "tp4" > gpurun_out/spc_tests4.log 2>&1; echo "tests chunks=4 rc $?"; tail -2 gpurun_out/spc_tests4.log
i=0
for c in 1 2 4 1 2; do
  i=$((i+1))
  GPTB200_SP_FWD_CHUNKS=$c GPTB200_TIMEOUT_S=200 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800+i)) bench.py --gpus 4 --workload ${W:-gpt-22b-tp4} --no-cpu-baseline --steps ${STEPS:-3} --warmup 2 > gpurun_out/spc_b_${i}_c$c.log 2>&1
  echo "chunks $c rc $?: $(tail -1 gpurun_out/spc_b_${i}_c$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), d["ms_per_step"], d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"],1) for k,v in d["kernels"].items() if v["ms_per_step"]})' 2>&1 | tail -1)"
done
