mkdir -p gpurun_out
TAG=f2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config1_matvec or hf_small or config2_sampled or direct_all or ragged or large_config" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 300 python tools/stage_times.py --config 2 > gpurun_out/stages_$TAG.json 2>&1
timeout 300 python tools/profile_matvec.py --config 2 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 90 --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_matvec.py --config 2 > gpurun_out/ncu_$TAG.log 2>&1
N=$(python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_f2.csv')) if len(r)>10 and r[0].isdigit()]
print(len(rows)//3 if rows else 22)
PY
)
timeout 1500 ncu --set full --clock-control none --import-source on -s $((2*N)) -c $N -o gpurun_out/prof_full_$TAG python tools/profile_matvec.py --config 2 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 1500 python tools/config5.py --cfg 5 --tc 1 --no-oracle > gpurun_out/cfg5_tc1_$TAG.json 2> gpurun_out/cfg5_tc1_$TAG.err
echo done
