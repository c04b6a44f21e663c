#!/bin/bash
# candidate builds vs the previous build on one box: GPU step/kernel tests (lib), then the 1.4B bench for
# each library in $LIBS (default: lib lib_old lib), all on the same box
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/ab_tests.log
i=0
for lib in ${LIBS:-lib lib_old lib}; do
  i=$((i+1))
  GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so timeout 400 python bench.py --no-cpu-baseline --steps ${STEPS:-10} --warmup 3 $EXTRA > gpurun_out/ab_bench_${i}_$lib.json 2> gpurun_out/ab_bench_${i}_$lib.err
  echo "$lib rc $?: $(tail -1 gpurun_out/ab_bench_${i}_$lib.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), d["ms_per_step"], d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"],1) for k,v in d["kernels"].items() if v["ms_per_step"]})' 2>&1 | tail -1)"
done
