#!/bin/bash
# full GPU suite + default bench + launch list of the bench's kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rP --durations=30 > gpurun_out/r02n_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02n_pytest.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
echo "bench rc=$?" >> gpurun_out/r02n_bench.err
tail -3 gpurun_out/r02n_pytest.log
