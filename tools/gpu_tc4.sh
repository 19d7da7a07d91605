mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core or config1_matvec or config2_sampled or large_config" > gpurun_out/pytest_tc4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc4.log
for tc in 0 2 1; do timeout 600 python tools/stage_times.py --config 3 --tc $tc >> gpurun_out/stages_tc4.jsonl 2>> gpurun_out/stages_tc4.err; done
timeout 300 python tools/profile_matvec.py --config 4 --tc 1 --warmup 0 --steps 1 > gpurun_out/plain_tc4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_xlate_tc" -s 0 -c 3 -o gpurun_out/prof_tc4_c4 python tools/profile_matvec.py --config 4 --tc 1 --warmup 0 --steps 1 > gpurun_out/ncu_tc4.log 2>&1
timeout 1500 python tools/config5.py --cfg 5 --tc 2 > gpurun_out/cfg5_tc4.json 2> gpurun_out/cfg5_tc4.err
echo done
