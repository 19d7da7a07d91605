#!/bin/bash
# k_xlate_bf: parity vs the CUDA-core translations, then A/B on configs 4 and 5
timeout 300 python tools/xbf_check.py --mesh 4 > gpurun_out/xbf_check.log 2>&1; echo "rc $?" >> gpurun_out/xbf_check.log
timeout 300 python tools/xbf_check.py --config 2 >> gpurun_out/xbf_check.log 2>&1; echo "rc $?" >> gpurun_out/xbf_check.log
cat gpurun_out/xbf_check.log
if grep -q "rel_l2_xbf_vs_cuda_core" gpurun_out/xbf_check.log; then
  timeout 600 python tools/ab_options.py --config 4 --steps 30 --variants '{}' '{"tensor_cores": 5}' > gpurun_out/ab_xbf4.jsonl 2> gpurun_out/ab_xbf4.err
  timeout 900 python tools/ab_options.py --config 5 --steps 10 --variants '{}' '{"tensor_cores": 5}' > gpurun_out/ab_xbf5.jsonl 2> gpurun_out/ab_xbf5.err
  python -c "
import json
for fn in ('gpurun_out/ab_xbf4.jsonl','gpurun_out/ab_xbf5.jsonl'):
  for l in open(fn):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n}, 'rel',d['rel_vs_first'])
"
fi
