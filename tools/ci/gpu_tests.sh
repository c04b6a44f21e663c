#!/bin/bash
# GPU test selection on one box: GPU_TESTS (pytest node ids / -k expressions) -> gpurun_out/<tag>.log
mkdir -p gpurun_out
tag=${TAG:-tests}
timeout ${TEST_TIMEOUT:-2400} python -m pytest -m gpu -q -s ${GPU_TESTS:-tests} > gpurun_out/$tag.log 2>&1
echo "pytest rc $?" >> gpurun_out/$tag.log
tail -40 gpurun_out/$tag.log
