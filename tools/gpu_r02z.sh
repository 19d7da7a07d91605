#!/bin/bash
# k_xlate_bf ring-size cap (co-residency with the near field) on configs 2-4
for c in 2 3 4; do
timeout 600 python tools/ab_options.py --config $c --steps 30 --variants '{}' '{"tensor_cores": 5}' \
  '{"tensor_cores": 5, "_env": {"FDA_XBF_SMEM_KB": 140}}' '{"tensor_cores": 5, "_env": {"FDA_XBF_SMEM_KB": 100}}' \
  '{"tensor_cores": 5, "_env": {"FDA_XBF_SMEM_KB": 72}}' > gpurun_out/ab_xbfs$c.jsonl 2> gpurun_out/ab_xbfs$c.err
done
python -c "
import json
for c in (2,3,4):
  for l in open(f'gpurun_out/ab_xbfs{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], d['env'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n}, 'rel',d['rel_vs_first'])
"
