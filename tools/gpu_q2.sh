mkdir -p gpurun_out
TAG=${1:-q2}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config1_matvec or hf_small or config2_sampled or direct_all or ragged or tensor_core or sharded or large_config" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for c in 2 3 4; do timeout 600 python tools/stage_times.py --config $c >> gpurun_out/stages_$TAG.jsonl 2>> gpurun_out/stages_$TAG.err; done
timeout 1500 python tools/config5.py --cfg 5 --no-oracle > gpurun_out/cfg5_$TAG.json 2> gpurun_out/cfg5_$TAG.err
echo done
