#!/bin/bash
# Debug a multi-GPU parity layout: runs tests/mp_worker.py ranks directly with a short timeout and
# prints each rank's output tail. $1 = json cfg, $2 = world size.
cfg=$1
world=$2
out=$(mktemp -d)
export NCCL_DEBUG=${NCCL_DEBUG:-WARN}
pids=()
for r in $(seq 0 $((world - 1))); do
  timeout -s ABRT 90 python -X faulthandler tests/mp_worker.py --cfg "$cfg" --rank $r --world $world --out $out \
    > $out/log$r 2>&1 &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; echo "exit $?"; done
for r in $(seq 0 $((world - 1))); do echo "=== rank $r"; tail -40 $out/log$r; done
