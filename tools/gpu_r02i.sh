#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rP -k "sharded" > gpurun_out/r02i_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02i_pytest.log
timeout 300 python tools/profile_matvec.py --config 4 --warmup 2 --steps 1 > gpurun_out/r02i_plain.log 2>&1 || exit 1
L=$(grep -o "launches_per_matvec [0-9]*" gpurun_out/r02i_plain.log | awk '{print $2}')
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_(gather|near|s2m|xlate|m2l|split|l2t|scatter)" -s $((2*L)) -c $L -o gpurun_out/r02i_full_c4 \
  python tools/profile_matvec.py --config 4 --warmup 2 --steps 1 > gpurun_out/r02i_ncu.log 2>&1
echo "ncu rc=$? launches=$L" >> gpurun_out/r02i_ncu.log
tail -3 gpurun_out/r02i_pytest.log
