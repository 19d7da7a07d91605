#!/bin/bash
# round-2 GPU check: full -m gpu suite + default bench (config 4 + configs 2/3)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
nproc >> gpurun_out/r02a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/r02a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a_pytest.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
echo "bench rc=$?" >> gpurun_out/r02a_bench.err
tail -5 gpurun_out/r02a_pytest.log
