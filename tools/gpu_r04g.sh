#!/bin/bash
# (experiment: needs profiles/r04_leaf_loop_experiment.patch applied to csrc/ and a rebuild)
# A/B: register-pipelined looping leaf kernels k_leaf_loop (FDA_LEAF_LOOP=0: the CTA-per-leaf kernels), then the GPU suite
out=gpurun_out/r04_ab_leaf_loop.jsonl; : > $out
for cfg in 2 4 5; do
  for st in 0 1; do
    FDA_LEAF_LOOP=$st timeout -k 10 300 python tools/stage_times.py --config $cfg --reps 20 | sed "s/^{/{\"leaf_loop\": $st, /" >> $out
    echo "cfg $cfg loop $st rc $?"
  done
done
cat $out
timeout -k 10 1100 python -m pytest tests -m gpu -x -q > gpurun_out/r04_pytest_gpu_loop.log 2>&1; tail -3 gpurun_out/r04_pytest_gpu_loop.log
