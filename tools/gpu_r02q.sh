#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -rP -x -k "tensor_core_fused" > gpurun_out/r02q_pytest.log 2>&1
rc=$?; echo "pytest rc=$rc" >> gpurun_out/r02q_pytest.log; [ $rc -eq 0 ] || exit 1
for c in 4 2; do
  timeout 300 python tools/ab_options.py --config $c --steps 20 --variants '{}' > gpurun_out/r02q_ab${c}_td.jsonl 2>> gpurun_out/r02q_ab.err
  FDA_M2L_DRAIN=0 timeout 300 python tools/ab_options.py --config $c --steps 20 --variants '{}' > gpurun_out/r02q_ab${c}_row.jsonl 2>> gpurun_out/r02q_ab.err
done
tail -2 gpurun_out/r02q_pytest.log
