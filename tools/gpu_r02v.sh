#!/bin/bash
# persistent near field (co-residency) on config 4; blocked M2L task order on config 5
python tools/ab_options.py --config 4 --steps 30 --variants '{}' \
  '{"_env": {"FDA_NEAR_PERSIST": 4}}' \
  '{"_env": {"FDA_NEAR_PERSIST": 3}}' \
  '{"_env": {"FDA_NEAR_PERSIST": 2, "FDA_M2L_SMEM_KB": 128}}' \
  '{"_env": {"FDA_NEAR_PERSIST": 3, "FDA_M2L_SMEM_KB": 100}}' \
  '{"_env": {"FDA_M2L_ORDER": "blocked"}}' > gpurun_out/ab_v4.jsonl 2> gpurun_out/ab_v4.err
python tools/ab_options.py --config 5 --steps 10 --variants '{}' \
  '{"_env": {"FDA_M2L_ORDER": "blocked"}}' \
  '{"_env": {"FDA_M2L_ORDER": "blocked", "FDA_M2L_BLOCK": 4}}' > gpurun_out/ab_v5.jsonl 2> gpurun_out/ab_v5.err
tail -3 gpurun_out/ab_v4.err gpurun_out/ab_v5.err
