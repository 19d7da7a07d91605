# reading C25 (α = −i/k): GPU parity suite, Table 2 with N_it, point-source workload
TAG=${1:-c25}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python tools/table2.py --nmin 3 --nmax 8 --eps 1e-3 > gpurun_out/table2_e3_$TAG.jsonl 2>&1
timeout 900 python tools/table2.py --nmin 3 --nmax 8 --eps 1e-4 > gpurun_out/table2_e4_$TAG.jsonl 2>&1
timeout 600 python tools/point_source.py > gpurun_out/point_source_$TAG.jsonl 2>&1
timeout 300 python tools/alpha_sign.py --config 4 > gpurun_out/alpha_sign_c4_$TAG.jsonl 2>&1
echo done
