#!/bin/bash
# Round 3a: TMA bulk-reduce drain in k_m2l_bf / k_xlate_bf — parity of the tensor-core kernels,
# then config-4 bench A/B against the RED.128 drain (FDA_DRAIN_RED=1), config-2/3 in the same lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "bf16 or tensor_core or config2 or large_config or sharded or device_build" \
  > gpurun_out/r03a_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r03a_pytest.log
for mode in 0 1; do
  FDA_DRAIN_RED=$mode timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r03a_bench_red$mode.json 2> gpurun_out/r03a_bench_red$mode.err
  echo "bench red=$mode rc=$?"
done
python - << 'PY'
import json
for m in (0, 1):
    try:
        d = json.loads(open(f"gpurun_out/r03a_bench_red{m}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(m, "no line", e); continue
    k = d["kernels"]
    print(f"red={m}: matvec {d['value']:.4f} ms, k_m2l_tcw(bf) {k['k_m2l_tcw']['ms']:.4f}, k_xlate_bf {k['k_xlate_bf']['ms']:.4f}, "
          f"near {k['k_near']['ms']:.4f}, cfg2 {d['other_configs']['config2']['matvec_ms']}, cfg3 {d['other_configs']['config3']['matvec_ms']}")
PY
