#!/bin/bash
# 4-GPU box: multi-GPU parity suite, then the multi-GPU bench lines
TAG=${TAG:-mgf} bash tools/ci/multigpu.sh
TAG=${TAG:-mgf}_b bash tools/ci/bench4.sh
