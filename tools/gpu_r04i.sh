#!/bin/bash
# final bench line of the round-4 code, then ncu --set full of the leaf kernels (config 4)
timeout 400 python bench.py --steps 50 --warmup 5 > gpurun_out/r04_bench_config4_final.json 2> gpurun_out/r04_bench_final.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r04_bench_config4_final.json
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash tools/gpu_ncu_k.sh r04_leaf_final 'k_s2m|k_l2t' 0 2 4
ncu -i gpurun_out/r04_leaf_final.ncu-rep --page raw --csv > gpurun_out/r04_leaf_final.csv 2>/dev/null; rm -f gpurun_out/r04_leaf_final.ncu-rep
