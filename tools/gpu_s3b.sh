# session 3 (after reading C25): Table 1 analogue (p_eq), Table 2 last row, config 3/4 stage times, bench
TAG=${1:-s3b}
mkdir -p gpurun_out
for p in 4 5 6 8; do timeout 600 python tools/table2.py --nmin 8 --nmax 8 --eps 1e-3 --p-eq $p; done > gpurun_out/table1_peq_$TAG.jsonl 2>&1
timeout 1200 python tools/table2.py --nmin 9 --nmax 9 --eps 1e-3 > gpurun_out/table2_n9_$TAG.jsonl 2>&1
for c in 3 4; do timeout 600 python tools/stage_times.py --config $c; done > gpurun_out/stages34_$TAG.jsonl 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo done
