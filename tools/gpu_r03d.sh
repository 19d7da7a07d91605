#!/bin/bash
# Round 3d: expanded q²/s near kernel (default) vs the difference form (FDA_NEAR_DIFF=1):
# GPU suite with the default, then stage times of configs 2 and 4 for both forms
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r03d_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r03d_pytest.log
grep -h "rel-L2\|rel_l2\|err" gpurun_out/r03d_pytest.log | head -5
for c in 2 4; do
  for m in 1 0; do
    FDA_NEAR_DIFF=$m timeout 300 python tools/stage_times.py --config $c --reps 20 | sed "s/^/diff=$m /"
  done
done > gpurun_out/r03d_stage.log 2>&1
cat gpurun_out/r03d_stage.log
