#!/bin/bash
# 4-GPU box: bench lines of the multi-GPU layouts (each its own torchrun launch and master port).
mkdir -p gpurun_out
tag=${TAG:-b4}
port=29600
run() {  # name ngpus extra-args...
  local name=$1 n=$2; shift 2; port=$((port + 1))
  GPTB200_TIMEOUT_S=300 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n "$@" > gpurun_out/${tag}_$name.json 2> gpurun_out/${tag}_$name.err
  echo "$name rc $?"; python - "$name" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/{sys.argv[0] if False else ''}".strip() or "/dev/null").read())
except Exception:
    pass
PY
  tail -c 400 gpurun_out/${tag}_$name.json; echo
}
run dp2 2 --steps 10 --warmup 3
run dp4 4 --steps 10 --warmup 3
run 22b_tp4 4 --workload gpt-22b-tp4 --steps 3 --warmup 2
run 175b_tp2pp2 4 --workload gpt-175b-slice-tp2pp2 --steps 3 --warmup 2
run 175b_tp2pp2_v2 4 --workload gpt-175b-slice-tp2pp2 --interleave 2 --steps 3 --warmup 2
run 175b_tp4 4 --workload gpt-175b-slice-tp4 --steps 3 --warmup 2
run 1t_tp4 4 --workload gpt-1t-slice-tp4 --steps 3 --warmup 2
