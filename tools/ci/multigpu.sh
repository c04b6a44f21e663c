#!/bin/bash
# Multi-GPU box call: the multi-GPU parity suite, then the 1T-slice TP4 checkpointed bench looped
# back to back (the configuration whose SP kernels could deadlock before the grid caps).
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
tag=${TAG:-mg}
timeout ${TEST_TIMEOUT:-3000} python -m pytest tests/test_multigpu.py -m gpu -q -s ${MG_TESTS:-} > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log
tail -30 gpurun_out/${tag}_pytest.log
if [ "$N" -ge 4 ] && [ -n "${LOOP_1T:-}" ]; then
  for i in $(seq 1 ${LOOP_1T}); do
    GPTB200_TIMEOUT_S=240 timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port $((29500 + i)) bench.py --gpus 4 --workload gpt-1t-slice-tp4 \
      --steps ${STEPS_1T:-5} --warmup 2 --no-cpu-baseline > gpurun_out/${tag}_1t_$i.json 2> gpurun_out/${tag}_1t_$i.err
    echo "1t loop $i rc $?"
    tail -c 600 gpurun_out/${tag}_1t_$i.json
  done
fi
if [ -n "${NCU_ATTN:-}" ]; then
  python tools/run_attn_shape.py 1 2048 40 160 bwd 2 && python tools/run_attn_shape.py 8 2048 16 128 bwd 2 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fa_bwd -c 2 -o gpurun_out/${NCU_ATTN}_hd160 \
     python tools/run_attn_shape.py 1 2048 40 160 bwd 2 > gpurun_out/${NCU_ATTN}_hd160.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fa_bwd -c 2 -o gpurun_out/${NCU_ATTN}_hd128 \
     python tools/run_attn_shape.py 8 2048 16 128 bwd 2 > gpurun_out/${NCU_ATTN}_hd128.log 2>&1
  echo "ncu rc $?"
fi
