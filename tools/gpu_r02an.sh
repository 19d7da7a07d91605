#!/bin/bash
# ncu --set full of one config-4 matvec (NVTX "fda_matvec"), then the k_xlate_bf share A/B and the config-5 run
mkdir -p gpurun_out
R=/tmp/r02b_full_c4_$$
timeout 1500 ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "fda_matvec/" -c 51 -o $R \
  python tools/profile_matvec.py --config 4 --warmup 0 --steps 1 > /tmp/ncu_full_c4_$$.log 2>&1; echo "ncu full rc=$?"
tail -2 /tmp/ncu_full_c4_$$.log
python tools/ncu_summary.py $R.ncu-rep gpurun_out/r02b_full_c4.json --label "config4 one matvec (r02 final, NVTX fda_matvec)" > gpurun_out/r02b_summary.log 2>&1; echo "summary rc=$?"
rm -f $R.ncu-rep
bash tools/gpu_r02am.sh
