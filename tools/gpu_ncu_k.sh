# ncu --set full of selected kernels of the first profiled matvec (after a plain run)
TAG=$1; REGEX=$2; SKIP=${3:-0}; CNT=${4:-4}; CFG=${5:-2}
mkdir -p gpurun_out
timeout 300 python tools/profile_matvec.py --config $CFG --warmup 0 --steps 1 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$REGEX" -s $SKIP -c $CNT -o gpurun_out/$TAG \
  python tools/profile_matvec.py --config $CFG --warmup 0 --steps 1 > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"
