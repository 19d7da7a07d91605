#!/bin/bash
# co-residency sweep of the config-4 graph matvec: near-field priority, k_m2l_bf ring size and grid
set -x
python tools/ab_options.py --config 4 --steps 30 --variants '{}' \
  '{"_env": {"FDA_NEAR_PRIO": "hi"}}' \
  '{"_env": {"FDA_M2L_SMEM_KB": 160}}' \
  '{"_env": {"FDA_M2L_SMEM_KB": 120}}' \
  '{"_env": {"FDA_M2L_GRID_PCT": 50}}' \
  '{"_env": {"FDA_M2L_GRID_PCT": 75, "FDA_M2L_SMEM_KB": 160}}' \
  '{"_env": {"FDA_NEAR_PRIO": "hi", "FDA_M2L_SMEM_KB": 120}}' > gpurun_out/ab_cores4.jsonl 2> gpurun_out/ab_cores4.err
tail -3 gpurun_out/ab_cores4.err
cat gpurun_out/ab_cores4.jsonl | cut -c1-400
