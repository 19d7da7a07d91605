#!/bin/bash
# k_m2l_bf for factored K̃ with r ≤ 48 (was 32): parity, then configs 4 and 5
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused_m2l or config2_sampled or large_config" > gpurun_out/pt_r48.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r48.log
tail -2 gpurun_out/pt_r48.log
for c in 4 3; do
timeout 600 python tools/ab_options.py --config $c --steps 30 --variants '{}' > gpurun_out/ab_r48_$c.jsonl 2> gpurun_out/ab_r48_$c.err
done
timeout 900 python tools/ab_options.py --config 5 --steps 10 --variants '{}' > gpurun_out/ab_r48_5.jsonl 2> gpurun_out/ab_r48_5.err
python -c "
import json
for c in (4,3,5):
  for l in open(f'gpurun_out/ab_r48_{c}.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n})
"
