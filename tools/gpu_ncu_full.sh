# one full matvec of a config under ncu --set full (after a plain run of the same command)
CFG=${1:-2}
OUT=${2:-prof_full_c$CFG}
mkdir -p gpurun_out
timeout 300 python tools/profile_matvec.py --config $CFG > gpurun_out/plain_$OUT.log 2>&1 || exit 1
L=$(grep -o "launches_per_matvec [0-9]*" gpurun_out/plain_$OUT.log | awk '{print $2}')
timeout 1500 ncu --set full --clock-control none --import-source on -s $((2*L)) -c $L -o gpurun_out/$OUT \
  python tools/profile_matvec.py --config $CFG > gpurun_out/ncu_$OUT.log 2>&1
echo "rc=$? launches=$L"
