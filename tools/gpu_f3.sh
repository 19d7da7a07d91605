mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "eps_sweep or tensor_core or sharded" > gpurun_out/pytest_f3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f3.log
bash tools/gpu_ncu_full.sh 2 prof_full_f3
echo done
