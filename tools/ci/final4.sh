#!/bin/bash
# Final-build 4-GPU check: multi-GPU parity at the BASELINE widths, then the TP / DP bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "22b_width or 175b_width or 1t_width or config1 or dp2_zero1" > gpurun_out/f4_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/f4_tests.log
i=0
for w in "gpt-22b-tp4" "gpt-175b-slice-tp4" "gpt-1.4b"; do
  i=$((i+1))
  GPTB200_TIMEOUT_S=200 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29950+i)) bench.py --gpus 4 --workload $w --no-cpu-baseline --steps ${STEPS:-5} --warmup 3 > gpurun_out/f4_b_$w.json 2> gpurun_out/f4_b_$w.err
  echo "$w rc $?: $(tail -1 gpurun_out/f4_b_$w.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), round(d["value"]), d["ms_per_step"], d["config"]["parallelism"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
done
