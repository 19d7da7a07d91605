#!/bin/bash
# locality (blocked) order of the translation tasks on config 5: k_xlate_tc (default) and k_xlate_bf
timeout 1500 python tools/ab_options.py --config 5 --steps 10 --variants '{}' '{"_env": {"FDA_XLATE_BLOCK": 1}}' \
  '{"_env": {"FDA_XLATE_BLOCK": 2}}' '{"tensor_cores": 5}' '{"tensor_cores": 5, "_env": {"FDA_XLATE_BLOCK": 1}}' \
  '{"tensor_cores": 5, "_env": {"FDA_XLATE_BLOCK": 2}}' > gpurun_out/ab_blk5.jsonl 2> gpurun_out/ab_blk5.err
tail -2 gpurun_out/ab_blk5.err
python -c "
import json
for l in open('gpurun_out/ab_blk5.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], d['env'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n}, 'rel',d['rel_vs_first'])
"
