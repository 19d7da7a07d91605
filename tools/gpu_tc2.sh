mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_tc2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc2.log
for c in 2 3; do for tc in 0 1 2; do timeout 600 python tools/stage_times.py --config $c --tc $tc >> gpurun_out/stages_tc2.jsonl 2>> gpurun_out/stages_tc2.err; done; done
echo done
