#!/bin/bash
# split near field: P persistent near CTAs per SM concurrent with the far field, Q more after it
python tools/ab_options.py --config 4 --steps 30 --variants '{}' \
  '{"_env": {"FDA_NEAR_PERSIST": 2, "FDA_NEAR_SPLIT": 2, "FDA_M2L_SMEM_KB": 128}}' \
  '{"_env": {"FDA_NEAR_PERSIST": 2, "FDA_NEAR_SPLIT": 2, "FDA_M2L_SMEM_KB": 120}}' \
  '{"_env": {"FDA_NEAR_PERSIST": 1, "FDA_NEAR_SPLIT": 3, "FDA_M2L_SMEM_KB": 170}}' \
  '{"_env": {"FDA_NEAR_PERSIST": 2, "FDA_NEAR_SPLIT": 2, "FDA_M2L_SMEM_KB": 128, "FDA_NEAR_PRIO": "hi"}}' \
  '{"_env": {"FDA_NEAR_PERSIST": 3, "FDA_NEAR_SPLIT": 1, "FDA_M2L_SMEM_KB": 80}}' > gpurun_out/ab_w4.jsonl 2> gpurun_out/ab_w4.err
tail -3 gpurun_out/ab_w4.err
python -c "
import json
for l in open('gpurun_out/ab_w4.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['env'], 'mv',d['matvec_ms'], 'near_live',d['near_live_ms'], 'm2l',k.get('k_m2l_tcw'), 'near',k.get('k_near'), 'rel',d['rel_vs_first'])
"
