#!/bin/bash
# One GPU box call: environment facts, the GPU test suite, the drop-in search on the GPU.
mkdir -p gpurun_out
{ nproc; free -g | head -2; lscpu | grep "Model name"; nvidia-smi -L; } > gpurun_out/env.txt 2>&1
python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
python -m pytest tests/test_dropin.py -m gpu -q -s > gpurun_out/dropin_gpu.log 2>&1; echo "dropin rc $?" >> gpurun_out/dropin_gpu.log
tail -5 gpurun_out/dropin_gpu.log
cat gpurun_out/env.txt
