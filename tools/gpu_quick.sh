# quick GPU round-trip: key parity tests, stage times, bench (config 2), launch list
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config1_matvec or hf_small or config2_sampled or direct_all or ragged or rhs_apply" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python tools/stage_times.py --config 2 > gpurun_out/stages_$TAG.json 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 300 python tools/profile_matvec.py --config 2 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 90 --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_matvec.py --config 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "done"
