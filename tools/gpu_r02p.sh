#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for g in 1 0.3 0.1; do
  for c in 4 3 2; do
    FDA_TC_MIN_GFLOP=$g timeout 600 python tools/ab_options.py --config $c --steps 20 --variants '{}' > gpurun_out/r02p_ab${c}_$g.jsonl 2>> gpurun_out/r02p_ab.err
  done
done
ls gpurun_out
