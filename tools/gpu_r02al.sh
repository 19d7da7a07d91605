#!/bin/bash
# k_xlate_bf with two CTAs per SM (FDA_XBF_CTAS=2): parity, then configs 4 and 5
FDA_XBF_CTAS=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "translations_bf16" > gpurun_out/pt_xbf2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_xbf2.log
tail -2 gpurun_out/pt_xbf2.log
if grep -q "pytest rc=0" gpurun_out/pt_xbf2.log; then
timeout 600 python tools/ab_options.py --config 4 --steps 30 --variants '{}' '{"_env": {"FDA_XBF_CTAS": 2}}' '{"tensor_cores": 5, "_env": {"FDA_XBF_CTAS": 2}}' > gpurun_out/ab_x2c4.jsonl 2> gpurun_out/ab_x2c4.err
timeout 600 python tools/ab_options.py --config 3 --steps 30 --variants '{"tensor_cores": 5}' '{"tensor_cores": 5, "_env": {"FDA_XBF_CTAS": 2}}' > gpurun_out/ab_x2c3.jsonl 2> gpurun_out/ab_x2c3.err
timeout 900 python tools/ab_options.py --config 5 --steps 10 --variants '{}' '{"_env": {"FDA_XBF_CTAS": 2}}' > gpurun_out/ab_x2c5.jsonl 2> gpurun_out/ab_x2c5.err
python -c "
import json
for c in (4,3,5):
  for l in open(f'gpurun_out/ab_x2c{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], d['env'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n}, 'rel',d['rel_vs_first'])
"
fi
