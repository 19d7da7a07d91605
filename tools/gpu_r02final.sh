#!/bin/bash
# round-2 final evidence: GPU suite, bench line, ncu launch list of the bench command, ncu --set full of one config-4 matvec
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest_gpu.log
tail -3 gpurun_out/final_pytest_gpu.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 1 > gpurun_out/final_ncu_bench.log 2>&1; echo "ncu list rc=$?"
bash tools/gpu_ncu_full.sh 4 final_full_c4
python tools/ncu_summary.py gpurun_out/final_full_c4.ncu-rep gpurun_out/final_full_c4.json --label "config4 one matvec (r02 final)" > /dev/null 2>&1; echo "summary rc=$?"
