mkdir -p gpurun_out
for c in 3 4 5; do timeout 1500 python tools/config5.py --cfg $c > gpurun_out/cfg${c}.json 2> gpurun_out/cfg${c}.err; echo "cfg $c rc=$?"; done
echo done
