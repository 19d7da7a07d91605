#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rP -k "tensor_core_fused" > gpurun_out/r02l_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02l_pytest.log
timeout 1200 python tools/ab_options.py --config 4 --variants '{}' > gpurun_out/r02l_ab4.jsonl 2> gpurun_out/r02l_ab4.err
timeout 900 python tools/ab_options.py --config 2 --variants '{}' > gpurun_out/r02l_ab2.jsonl 2> gpurun_out/r02l_ab2.err
tail -3 gpurun_out/r02l_pytest.log
