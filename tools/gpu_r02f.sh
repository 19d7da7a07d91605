#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rP -k "device_build or config2_sampled or tensor_core_fused" > gpurun_out/r02f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f_pytest.log
FDA_VERBOSE=2 timeout 900 python tools/build_times.py --configs 5 4 > gpurun_out/r02f_build.jsonl 2> gpurun_out/r02f_build.err
tail -3 gpurun_out/r02f_pytest.log
