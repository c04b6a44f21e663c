#!/bin/bash
# two-rank smoke of the session (debug): $1 = library path
export GPTB200_LIB=$1
export NCCL_DEBUG=WARN
timeout 200 python -X faulthandler -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 2 --warmup 1 --workload gpt-tiny --no-profile 2>&1 | grep -v "^\s*$" | tail -25
