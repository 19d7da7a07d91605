#!/bin/bash
# k_m2l_bf with ≤ 96 registers and a capped ring: co-residency with two near-field CTAs per SM
for c in 4 3; do
timeout 600 python tools/ab_options.py --config $c --steps 30 --variants '{}' '{"_env": {"FDA_M2L_SMEM_KB": 128}}' \
  '{"_env": {"FDA_M2L_SMEM_KB": 120}}' '{"_env": {"FDA_M2L_SMEM_KB": 100}}' '{"_env": {"FDA_M2L_SMEM_KB": 170}}' > gpurun_out/ab_m2lco$c.jsonl 2> gpurun_out/ab_m2lco$c.err
done
python -c "
import json
for c in (4,3):
  for l in open(f'gpurun_out/ab_m2lco{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['env'], 'mv',d['matvec_ms'], 'near_live', d['near_live_ms'], {n:v for n,v in k.items() if 'm2l' in n}, 'rel',d['rel_vs_first'])
"
