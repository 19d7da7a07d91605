#!/bin/bash
# ncu --set full of the two largest k_xlate_bf launches (config 5 M2M L7, L6) and one k_xlate_tc launch
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_xlate_bf" -c 2 -o gpurun_out/xbf5 \
  python tools/profile_matvec.py --config 5 --warmup 0 --steps 1 --tc 5 > gpurun_out/ncu_xbf5.log 2>&1
echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_xlate_tc" -c 1 -o gpurun_out/xtc5 \
  python tools/profile_matvec.py --config 5 --warmup 0 --steps 1 --tc 2 > gpurun_out/ncu_xtc5.log 2>&1
echo "rc=$?"
python tools/ncu_summary.py gpurun_out/xbf5.ncu-rep gpurun_out/xbf5_summary.json --label "config5 k_xlate_bf M2M L7/L6"
python tools/ncu_summary.py gpurun_out/xtc5.ncu-rep gpurun_out/xtc5_summary.json --label "config5 k_xlate_tc first"
tail -3 gpurun_out/ncu_xbf5.log
