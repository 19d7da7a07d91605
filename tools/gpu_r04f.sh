#!/bin/bash
# (experiment: needs profiles/r04_leaf_pipe_experiment.patch applied to csrc/ and a rebuild)
# ncu --set full of the leaf kernels at config 4: pipelined (k_leaf_pipe) and one-CTA-per-leaf (k_s2m / k_l2t)
bash tools/gpu_ncu_k.sh r04_leaf_pipe 'k_leaf_pipe' 0 2 4
FDA_LEAF_PIPE=0 bash tools/gpu_ncu_k.sh r04_leaf_cta 'k_s2m|k_l2t' 0 2 4
ls -la gpurun_out/*.ncu-rep
