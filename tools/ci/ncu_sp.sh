#!/bin/bash
# NVLink bytes of the fused SP LayerNorm kernels and the NVLS allreduce (ncu on rank 0, 4 GPUs)
mkdir -p gpurun_out
ncu --query-metrics 2>/dev/null | grep -iE "^nvl(rx|tx)__bytes" | head -5 > gpurun_out/ncu_sp_metrics.txt
for d in "6144 48" "25600 160"; do
  set -- $d
  HID=$1 GPTB200_TIMEOUT_S=120 timeout 300 python -m torch.distributed.run --no-python --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port $((29900 + RANDOM % 50)) bash tools/ci/ncu_rank0.sh --hidden $1 --heads $2 --iters 2 \
    > gpurun_out/ncu_sp_run_$1.log 2>&1
  echo "d=$1 rc $?"
done
