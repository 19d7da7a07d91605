#!/bin/bash
# round-2 final evidence: bench line, ncu launch list of the bench command, ncu --set full of one
# config-4 matvec (report kept in /tmp on the box; only its summary comes back), config-5 check
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 1 > /tmp/final_ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 300 python tools/profile_matvec.py --config 4 > /tmp/plain_c4.log 2>&1
L=$(grep -o "launches_per_matvec [0-9]*" /tmp/plain_c4.log | awk '{print $2}')
timeout 1500 ncu --set full --clock-control none --import-source on -s $((2*L)) -c $L -o /tmp/final_full_c4 \
  python tools/profile_matvec.py --config 4 > /tmp/ncu_full_c4.log 2>&1; echo "ncu full rc=$? launches=$L"
python tools/ncu_summary.py /tmp/final_full_c4.ncu-rep gpurun_out/final_full_c4.json --label "config4 one matvec (r02 final)" > gpurun_out/final_summary.log 2>&1; echo "summary rc=$?"
ls -la gpurun_out | head
