#!/bin/bash
# per-stage share threshold for k_xlate_bf at config 4 / 5, then the config-5 run (matvec, parity, solve)
timeout 900 python tools/ab_options.py --config 4 --steps 30 --variants '{}' '{"_env": {"FDA_XBF_MIN_SHARE": 64}}' \
  '{"_env": {"FDA_XBF_MIN_SHARE": 256}}' '{"_env": {"FDA_XBF_MIN_SHARE": 1000}}' > gpurun_out/ab_share4.jsonl 2> gpurun_out/ab_share4.err
python -c "
import json
for l in open('gpurun_out/ab_share4.jsonl'):
    d=json.loads(l); k=d['kernels_ms']; print(d['config'], d['env'], 'mv',d['matvec_ms'], {n:v for n,v in k.items() if 'xlate' in n or 'm2l' in n})
"
timeout 1500 python tools/config5.py --solve > gpurun_out/config5_final.json 2> gpurun_out/config5_final.err; echo "config5 rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/config5_final.json').read().strip().splitlines()[-1])
print({k:d[k] for k in ('N','build_s','matvec_ms','rel_l2_sampled','oracle_rows_s')}, d['stages_ms'], d['solve'])
"
