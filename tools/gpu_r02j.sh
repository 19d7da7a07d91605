#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rP -k "sharded" > gpurun_out/r02j_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02j_pytest.log
timeout 1200 python tools/ab_options.py --config 4 --variants '{}' '{"lr_tensor_cores": 1}' '{"tensor_cores": 1}' '{"tensor_cores": 1, "lr_tensor_cores": 1}' '{"m2l_bf16": 0}' > gpurun_out/r02j_ab4.jsonl 2> gpurun_out/r02j_ab4.err
timeout 900 python tools/ab_options.py --config 3 --variants '{}' '{"lr_tensor_cores": 1}' '{"tensor_cores": 1, "lr_tensor_cores": 1}' > gpurun_out/r02j_ab3.jsonl 2> gpurun_out/r02j_ab3.err
timeout 900 python tools/ab_options.py --config 2 --variants '{}' '{"lr_tensor_cores": 1}' '{"tensor_cores": 1, "lr_tensor_cores": 1}' > gpurun_out/r02j_ab2.jsonl 2> gpurun_out/r02j_ab2.err
tail -3 gpurun_out/r02j_pytest.log
