#!/bin/bash
# leaf kernels: stage times of configs 2/4/5 (baseline: profiles/r04_leaf_addr.jsonl), then the GPU suite
out=gpurun_out/r04_leaf_presync.jsonl; : > $out
for cfg in 2 4 5; do
  timeout -k 10 300 python tools/stage_times.py --config $cfg --reps 20 >> $out
done
cat $out
timeout -k 10 1100 python -m pytest tests -m gpu -x -q > gpurun_out/r04_pytest_gpu_presync.log 2>&1; tail -3 gpurun_out/r04_pytest_gpu_presync.log
