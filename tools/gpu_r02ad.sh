#!/bin/bash
# far field alone (near kernel skipped) vs the full graph matvec
for c in 4 3 2; do
timeout 600 python tools/ab_options.py --config $c --steps 30 --variants '{}' > gpurun_out/ab_far$c.jsonl 2>&1
FDA_SKIP_NEAR=1 timeout 600 python tools/ab_options.py --config $c --steps 30 --variants '{}' >> gpurun_out/ab_far$c.jsonl 2>&1
grep matvec_ms gpurun_out/ab_far$c.jsonl | cut -c1-200
done
