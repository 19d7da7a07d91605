mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v5.log
for c in 2 3 4; do timeout 600 python tools/stage_times.py --config $c >> gpurun_out/stages_v5.jsonl 2>> gpurun_out/stages_v5.err; done
timeout 1500 python tools/config5.py --cfg 5 > gpurun_out/cfg5_v5.json 2> gpurun_out/cfg5_v5.err
echo done
