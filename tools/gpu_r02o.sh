#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rP -k "hf_leaves or device_build" > gpurun_out/r02o_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02o_pytest.log
timeout 300 python tools/sanitize_small.py > gpurun_out/r02o_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/r02o_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/r02o_memcheck.log
timeout 600 python tools/ab_options.py --config 4 --variants '{}' > gpurun_out/r02o_ab4.jsonl 2> gpurun_out/r02o_ab4.err
tail -3 gpurun_out/r02o_pytest.log
