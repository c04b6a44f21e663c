#!/bin/bash
# 1-GPU box: GPU test suite, the default bench (driver command), the reference arm.
mkdir -p gpurun_out
tag=${TAG:-b1}
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
  tail -3 gpurun_out/${tag}_pytest.log
fi
timeout 900 python bench.py --gpus 1 --steps ${STEPS:-20} --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?"
tail -c 1500 gpurun_out/${tag}_bench.json
if [ -z "${SKIP_REF:-}" ]; then
  timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref rc $?"
  tail -c 800 gpurun_out/${tag}_ref.json
fi
