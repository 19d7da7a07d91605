#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/profile_matvec.py --config 4 --warmup 2 --steps 1 > gpurun_out/r02i_plain.log 2>&1 || exit 1
L=$(grep -o "launches_per_matvec [0-9]*" gpurun_out/r02i_plain.log | awk '{print $2}')
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_(gather|near|s2m|xlate|m2l|split|l2t|scatter)" -s $((2*L)) -c $L -o /tmp/r02i_full_c4 \
  python tools/profile_matvec.py --config 4 --warmup 2 --steps 1 > gpurun_out/r02i_ncu.log 2>&1
echo "ncu rc=$? launches=$L" >> gpurun_out/r02i_ncu.log
python tools/ncu_summary.py /tmp/r02i_full_c4.ncu-rep gpurun_out/r02i_summary_c4.json --label "config4 one matvec (r02)" >> gpurun_out/r02i_ncu.log 2>&1
ncu -i /tmp/r02i_full_c4.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null && python - <<'PY'
import csv, json
rows = list(csv.reader(open("/tmp/raw.csv")))
hdr = rows[0]
keep = [r for r in rows[2:] if len(r) == len(hdr) and ("m2l_bf" in r[hdr.index("Kernel Name")] or "k_near" in r[hdr.index("Kernel Name")])]
out = [{h: v for h, v in zip(hdr, r)} for r in keep[:3]]
json.dump(out, open("gpurun_out/r02i_raw_m2l_near.json", "w"))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_m2l_bf" -s 2 -c 1 -o gpurun_out/r02i_m2l_bf \
  python tools/profile_matvec.py --config 4 --warmup 2 --steps 1 > gpurun_out/r02i_ncu2.log 2>&1
ls -la gpurun_out
