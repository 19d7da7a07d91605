#!/bin/bash
# ncu evidence restricted to the matvec (NVTX range "fda_matvec"; the device build's kernels excluded):
# launch list of the bench command, and --set full of one config-4 matvec (report in /tmp on the box)
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fda_matvec/" -c 400 --csv \
  --log-file gpurun_out/r04_ncu_bench_launches.csv python bench.py --steps 2 --warmup 1 > /tmp/final_ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "fda_matvec/" -c 51 -o /tmp/final_full_c4 \
  python tools/profile_matvec.py --config 4 --warmup 0 --steps 1 > /tmp/ncu_full_c4.log 2>&1; echo "ncu full rc=$?"
tail -3 /tmp/ncu_full_c4.log
python tools/ncu_summary.py /tmp/final_full_c4.ncu-rep gpurun_out/r04_ncu_full_matvec_config4.json --label "config4 one matvec (r04 final)" > gpurun_out/r04_summary.log 2>&1; echo "summary rc=$?"
