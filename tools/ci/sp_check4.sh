#!/bin/bash
# 4-GPU: SP kernel A/B in isolation, TP parity tests, 22B / 175B TP4 bench (old vs new library)
NP=4 bash tools/ci/sp_ab.sh
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "tp2 or tp4 or config1" > gpurun_out/sp4_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/sp4_tests.log
i=0
for lib in lib lib_old; do
for w in "gpt-22b-tp4" "gpt-175b-slice-tp4"; do
  i=$((i+1))
  GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so GPTB200_TIMEOUT_S=300 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29650+i)) bench.py --gpus 4 --workload $w --no-cpu-baseline > gpurun_out/sp4_b$i.log 2>&1
  echo "$lib $w: $(tail -1 gpurun_out/sp4_b$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), round(d["value"]), d["ms_per_step"], d["config"]["parallelism"], d["clocks"]["sm_mhz"], d["kernels"]["tp_comm"]["ms_per_step"])' 2>&1 | tail -1)"
done; done
