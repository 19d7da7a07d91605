#!/bin/bash
# near-kernel CTA shape / unroll variants (FDA_NEAR_VARIANT) on configs 4 and 2
for c in 4 2; do
timeout 900 python tools/ab_options.py --config $c --steps 30 --variants '{}' '{"_env": {"FDA_NEAR_VARIANT": 1}}' '{"_env": {"FDA_NEAR_VARIANT": 2}}' \
 '{"_env": {"FDA_NEAR_VARIANT": 3}}' '{"_env": {"FDA_NEAR_VARIANT": 4}}' '{"_env": {"FDA_NEAR_VARIANT": 5}}' '{"_env": {"FDA_NEAR_VARIANT": 6}}' \
 '{"_env": {"FDA_NEAR_VARIANT": 7}}' '{"_env": {"FDA_NEAR_VARIANT": 8}}' > gpurun_out/ab_nv$c.jsonl 2> gpurun_out/ab_nv$c.err
done
python -c "
import json
for c in (4,2):
  for l in open(f'gpurun_out/ab_nv{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['env'], 'mv',d['matvec_ms'], 'near_live', d['near_live_ms'], 'near', k.get('k_near'), 'rel',d['rel_vs_first'])
"
