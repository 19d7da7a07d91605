mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ps.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ps.log
timeout 900 python tools/point_source.py > gpurun_out/point_source.jsonl 2> gpurun_out/point_source.err
for p in 3 4 5 6 8; do timeout 900 python tools/table2.py --nmin 8 --nmax 8 --eps 1e-3 --p-eq $p >> gpurun_out/table1_n8.jsonl 2>> gpurun_out/table1.err; done
echo done
