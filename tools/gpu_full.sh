# full GPU round: parity suite, bench (config 2), launch list, ncu --set full of one matvec
TAG=${1:-full}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 300 python tools/stage_times.py --config 2 > gpurun_out/stages_$TAG.json 2>&1
timeout 300 python tools/profile_matvec.py --config 2 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 90 --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_matvec.py --config 2 > gpurun_out/ncu_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -s 42 -c 21 -o gpurun_out/prof_full_$TAG python tools/profile_matvec.py --config 2 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "done"
