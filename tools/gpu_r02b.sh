#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rP -k "stage_times or sharded or general_complex or tensor_core_translations" > gpurun_out/r02b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
echo "bench rc=$?" >> gpurun_out/r02b_bench.err
tail -3 gpurun_out/r02b_pytest.log
