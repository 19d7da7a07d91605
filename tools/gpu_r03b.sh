#!/bin/bash
# Round 3b: GPU suite, config-4 bench line, build phase times of configs 4 and 5 (pair search per size
# class, range-finder level SVDs)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r03b_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r03b_pytest.log
timeout 600 python bench.py > gpurun_out/r03b_bench.json 2> gpurun_out/r03b_bench.err; echo "bench rc=$?"
FDA_VERBOSE=2 timeout 600 python tools/build_times.py --configs 4 5 > gpurun_out/r03b_build_times.log 2>&1; echo "build_times rc=$?"
python - << 'PY'
import json
d = json.loads(open("gpurun_out/r03b_bench.json").read().strip().splitlines()[-1])
print("matvec", d["value"], "e2e", d["e2e"]["value"], "build_s", d["build_s"], "rank", d["tree"]["rank"], "solve", d["solve"])
PY
grep "fda_build\]\|pair search\|engine_create\|config" gpurun_out/r03b_build_times.log
