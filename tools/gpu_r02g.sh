#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rP -k "tensor_core_fused or config2_sampled or device_build" > gpurun_out/r02g_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02g_pytest.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
FDA_VERBOSE=2 timeout 900 python tools/build_times.py --configs 5 > gpurun_out/r02g_build.jsonl 2> gpurun_out/r02g_build.err
tail -3 gpurun_out/r02g_pytest.log
