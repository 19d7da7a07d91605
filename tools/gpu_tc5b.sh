mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core or config1_matvec" > gpurun_out/pytest_tc5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc5.log
for c in 3 4; do for tc in 0 2 3; do timeout 600 python tools/stage_times.py --config $c --tc $tc >> gpurun_out/stages_tc5.jsonl 2>> gpurun_out/stages_tc5.err; done; done
for tc in 3 2; do timeout 1500 python tools/config5.py --cfg 5 --tc $tc --no-oracle >> gpurun_out/cfg5_tc5.jsonl 2>> gpurun_out/cfg5_tc5.err; done
echo done
