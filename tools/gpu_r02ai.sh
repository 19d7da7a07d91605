#!/bin/bash
# k_m2l_bf drain through TMA bulk f32 reductions: parity tests, then configs 2-5
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused_m2l or config2_sampled or bf16" > gpurun_out/pt_bulk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_bulk.log
tail -3 gpurun_out/pt_bulk.log
if grep -q "pytest rc=0" gpurun_out/pt_bulk.log; then
for c in 2 3 4; do
timeout 600 python tools/ab_options.py --config $c --steps 30 --variants '{}' > gpurun_out/ab_bulk$c.jsonl 2> gpurun_out/ab_bulk$c.err
done
timeout 900 python tools/ab_options.py --config 5 --steps 10 --variants '{}' > gpurun_out/ab_bulk5.jsonl 2> gpurun_out/ab_bulk5.err
python -c "
import json
for c in (2,3,4,5):
  for l in open(f'gpurun_out/ab_bulk{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n})
"
fi
