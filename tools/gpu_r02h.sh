#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rP -k "sharded" > gpurun_out/r02h_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02h_pytest.log
timeout 600 python tools/wx_lists.py --config 4 > gpurun_out/r02h_wx.json 2> gpurun_out/r02h_wx.err
timeout 300 python tools/profile_matvec.py --config 4 > gpurun_out/r02h_plain.log 2>&1 || exit 1
L=$(grep -o "launches_per_matvec [0-9]*" gpurun_out/r02h_plain.log | awk '{print $2}')
timeout 1500 ncu --set full --clock-control none --import-source on -s $((2*L)) -c $L -o gpurun_out/r02h_full_c4 \
  python tools/profile_matvec.py --config 4 > gpurun_out/r02h_ncu.log 2>&1
echo "ncu rc=$? launches=$L" >> gpurun_out/r02h_ncu.log
tail -3 gpurun_out/r02h_pytest.log
