#!/bin/bash
# shared-memory carveout of the CUDA-core kernels (co-residency of near and far field)
for c in 4 3 2; do
timeout 900 python tools/ab_options.py --config $c --steps 30 --variants '{}' '{"_env": {"FDA_CARVEOUT": 100}}' \
  '{"_env": {"FDA_CARVEOUT": 100, "FDA_M2L_SMEM_KB": 128}}' '{"_env": {"FDA_CARVEOUT": 100, "FDA_M2L_SMEM_KB": 170}}' \
  '{"tensor_cores": 5, "_env": {"FDA_CARVEOUT": 100}}' > gpurun_out/ab_cv$c.jsonl 2> gpurun_out/ab_cv$c.err
done
python -c "
import json
for c in (4,3,2):
  for l in open(f'gpurun_out/ab_cv{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], d['env'], 'mv',d['matvec_ms'], 'near_live', d['near_live_ms'], 'near', k.get('k_near'), 'rel',d['rel_vs_first'])
"
