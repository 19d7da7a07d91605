#!/bin/bash
# near/far overlap: graph vs eager streams, near priority
timeout 900 python tools/ab_options.py --config 4 --steps 30 --variants '{}' '{"use_graph": 0}' > gpurun_out/ab_eager4.jsonl 2> gpurun_out/ab_eager4.err
FDA_SKIP_NEAR=1 timeout 900 python tools/ab_options.py --config 4 --steps 30 --variants '{"use_graph": 0}' >> gpurun_out/ab_eager4.jsonl 2>> gpurun_out/ab_eager4.err
python -c "
import json
for l in open('gpurun_out/ab_eager4.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['options'], d['env'], 'mv',d['matvec_ms'], 'near_live', d['near_live_ms'])
"
