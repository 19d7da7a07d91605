mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "hf_leaves or eps_sweep or config1_matvec" > gpurun_out/pytest_hf.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_hf.log
echo done
