#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rP -k "device_build or config1 or config2_sampled or small_and_ragged or hf_ or rhs or pulsating or general" > gpurun_out/r02c_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02c_pytest.log
timeout 900 python tools/build_times.py --configs 4 5 > gpurun_out/r02c_build.jsonl 2> gpurun_out/r02c_build.err
echo "build rc=$?" >> gpurun_out/r02c_build.err
tail -3 gpurun_out/r02c_pytest.log
