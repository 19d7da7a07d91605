#!/bin/bash
timeout 300 python tools/xbf_check.py --mesh 4 > gpurun_out/xbf_check2.log 2>&1; echo "rc $?" >> gpurun_out/xbf_check2.log
timeout 300 python tools/xbf_check.py --config 2 >> gpurun_out/xbf_check2.log 2>&1; echo "rc $?" >> gpurun_out/xbf_check2.log
cat gpurun_out/xbf_check2.log | cut -c1-300
timeout 600 python tools/ab_options.py --config 4 --steps 30 --variants '{}' '{"tensor_cores": 5}' > gpurun_out/ab_xbf4.jsonl 2> gpurun_out/ab_xbf4.err
timeout 600 python tools/ab_options.py --config 3 --steps 30 --variants '{}' '{"tensor_cores": 5}' > gpurun_out/ab_xbf3.jsonl 2> gpurun_out/ab_xbf3.err
timeout 600 python tools/ab_options.py --config 2 --steps 30 --variants '{}' '{"tensor_cores": 5}' > gpurun_out/ab_xbf2.jsonl 2> gpurun_out/ab_xbf2.err
python -c "
import json
for fn in ('gpurun_out/ab_xbf2.jsonl','gpurun_out/ab_xbf3.jsonl','gpurun_out/ab_xbf4.jsonl'):
  for l in open(fn):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n}, 'rel',d['rel_vs_first'])
"
