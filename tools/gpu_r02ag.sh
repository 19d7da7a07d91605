#!/bin/bash
# new default (k_xlate_bf on large shared stages) on configs 2-5, then the GPU suite
for c in 2 3 4; do
timeout 600 python tools/ab_options.py --config $c --steps 30 --variants '{}' '{"tensor_cores": 5}' > gpurun_out/ab_def$c.jsonl 2> gpurun_out/ab_def$c.err
done
timeout 900 python tools/ab_options.py --config 5 --steps 10 --variants '{}' > gpurun_out/ab_def5.jsonl 2> gpurun_out/ab_def5.err
python -c "
import json
for c in (2,3,4,5):
  for l in open(f'gpurun_out/ab_def{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n}, 'rel',d['rel_vs_first'])
"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
