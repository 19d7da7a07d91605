mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core or config1_matvec" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
for c in 2 3; do for tc in 0 1; do timeout 600 python tools/stage_times.py --config $c --tc $tc >> gpurun_out/stages_tc.jsonl 2>> gpurun_out/stages_tc.err; done; done
echo done
