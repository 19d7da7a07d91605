#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_complex64 or config1" > gpurun_out/pt_c64.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_c64.log
tail -2 gpurun_out/pt_c64.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/final4_bench.json 2> gpurun_out/final4_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/final4_bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e'],'frac',round(d['roofline']['frac'],3))
"
