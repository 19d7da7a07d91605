mkdir -p gpurun_out
timeout 900 python tools/config5.py --cfg 4 --tc 1 > gpurun_out/cfg4_tc.json 2> gpurun_out/cfg4_tc.err; echo "cfg4 rc=$?"
timeout 1500 python tools/config5.py --cfg 5 --tc 1 > gpurun_out/cfg5_tc.json 2> gpurun_out/cfg5_tc.err; echo "cfg5 rc=$?"
echo done
