#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -rP -x -k "tensor_core_fused" > gpurun_out/r02m_pytest.log 2>&1
rc=$?
echo "pytest rc=$rc" >> gpurun_out/r02m_pytest.log
[ $rc -eq 0 ] || exit 1
timeout 300 python tools/ab_options.py --config 4 --steps 20 --variants '{}' > gpurun_out/r02m_ab4.jsonl 2> gpurun_out/r02m_ab4.err
timeout 300 python tools/profile_matvec.py --config 4 --warmup 2 --steps 1 > gpurun_out/r02m_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_m2l_bf" -s 2 -c 1 -o gpurun_out/r02m_m2l_bf \
  python tools/profile_matvec.py --config 4 --warmup 2 --steps 1 > gpurun_out/r02m_ncu.log 2>&1
tail -3 gpurun_out/r02m_pytest.log
