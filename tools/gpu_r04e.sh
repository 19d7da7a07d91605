#!/bin/bash
# (experiment: needs profiles/r04_leaf_pipe_experiment.patch applied to csrc/ and a rebuild)
# A/B: persistent pipelined leaf kernels k_leaf_pipe, second version (256 consumers, column-aligned chunks, 3 CTAs/SM)
out=gpurun_out/r04_ab_leaf_pipe2.jsonl; : > $out
for cfg in 2 4 5; do
  for st in 0 1; do
    FDA_LEAF_PIPE=$st timeout -k 10 300 python tools/stage_times.py --config $cfg --reps 20 | sed "s/^{/{\"leaf_pipe\": $st, /" >> $out
    echo "cfg $cfg pipe $st rc $?"
  done
done
cat $out
