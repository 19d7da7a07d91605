#!/bin/bash
# auto rule (k_xlate_bf on problems with >= 10 GFLOP of dense translations): configs 2-5, then bench
for c in 2 3 4; do
timeout 600 python tools/ab_options.py --config $c --steps 30 --variants '{}' '{"tensor_cores": 5}' > gpurun_out/ab_auto$c.jsonl 2> gpurun_out/ab_auto$c.err
done
timeout 900 python tools/ab_options.py --config 5 --steps 10 --variants '{}' > gpurun_out/ab_auto5.jsonl 2> gpurun_out/ab_auto5.err
python -c "
import json
for c in (2,3,4,5):
  for l in open(f'gpurun_out/ab_auto{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n}, 'rel',d['rel_vs_first'])
"
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.json
