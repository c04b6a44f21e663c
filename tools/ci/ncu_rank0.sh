#!/bin/bash
# torchrun --no-python target: rank 0 runs tools/bench_sp.py under ncu with single-pass NVLink metrics
# (no kernel replay, which would deadlock the cross-GPU barriers); the other ranks run it plainly.
if [ "$RANK" = "0" ]; then
  exec timeout 240 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum --clock-control none \
    -k regex:"sp_ln|nvls_allreduce" -c ${NCU_COUNT:-6} --csv --log-file gpurun_out/ncu_sp_${HID}.csv \
    python tools/bench_sp.py "$@"
else
  exec timeout 240 python tools/bench_sp.py "$@"
fi
