mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded or point_source or config1_matvec or hf_small" > gpurun_out/pytest_mg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mg.log
timeout 900 python tools/table2.py --nmin 3 --nmax 7 --eps 1e-3 > gpurun_out/table2_e3.jsonl 2> gpurun_out/table2_e3.err
timeout 900 python tools/table2.py --nmin 3 --nmax 7 --eps 1e-4 > gpurun_out/table2_e4.jsonl 2> gpurun_out/table2_e4.err
echo done
