i=0
for w in "gpt-1.4b" "gpt-22b-tp4" "gpt-22b-tp2" "gpt-175b-slice-tp4" "gpt-175b-slice-tp2pp2 --interleave 2" "gpt-1t-slice-tp4"; do
  i=$((i+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py --gpus 4 --workload $w --no-cpu-baseline > gpurun_out/b4_$i.log 2>&1
  echo "$w: $(tail -1 gpurun_out/b4_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["model_tflops_per_gpu"],1), round(d["value"]), d["ms_per_step"], d["config"]["parallelism"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
done
