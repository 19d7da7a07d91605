#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/devbuild_diff.py > gpurun_out/r02e_diff.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rP -k "sharded or device_build" > gpurun_out/r02e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
FDA_VERBOSE=2 timeout 900 python tools/build_times.py --configs 5 > gpurun_out/r02e_build.jsonl 2> gpurun_out/r02e_build.err
tail -3 gpurun_out/r02e_pytest.log
