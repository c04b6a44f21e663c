#!/bin/bash
# GEMM change A/B on one box: kernel tests, sustained GEMMs at the MBS-32 step shapes, then the 1.4B bench
# (lib = candidate, lib_old = previous build; bench order new, old, new)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -m gpu -x -q > gpurun_out/gab_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/gab_tests.log
for lib in lib lib_old; do
  echo "== $lib"; GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so SHAPES=mbs32 timeout 400 python tools/bench_gemm_sustained.py 2>&1 | grep "^ours"
done
for lib in lib lib_old lib; do
  GPTB200_LIB=$PWD/paper_2312_12705_b200/$lib/libtrainplan_b200.so timeout 400 python bench.py --no-cpu-baseline --steps ${STEPS:-10} --warmup 3 > gpurun_out/gab_bench_$lib.json 2> gpurun_out/gab_bench_$lib.err
  echo "$lib rc $?: $(tail -1 gpurun_out/gab_bench_$lib.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), d["ms_per_step"], d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"],1) for k,v in d["kernels"].items() if v["ms_per_step"]})' 2>&1 | tail -1)"
done
