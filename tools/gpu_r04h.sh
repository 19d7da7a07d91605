#!/bin/bash
# leaf kernels with pointer-increment addressing (baseline: the leaf_loop = 0 rows of profiles/r04_ab_leaf_loop.jsonl), then the GPU suite
out=gpurun_out/r04_leaf_addr.jsonl; : > $out
for cfg in 2 4 5; do
  timeout -k 10 300 python tools/stage_times.py --config $cfg --reps 20 >> $out
done
cat $out
timeout -k 10 1100 python -m pytest tests -m gpu -x -q > gpurun_out/r04_pytest_gpu_addr.log 2>&1; tail -3 gpurun_out/r04_pytest_gpu_addr.log
