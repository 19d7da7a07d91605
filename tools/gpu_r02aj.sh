#!/bin/bash
# device-resident pool and correction values (no download / re-upload): tests, then config 4/5 build times
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "device_build or config1 or rhs or pulsating or config2_sampled" > gpurun_out/pt_devres.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_devres.log
tail -3 gpurun_out/pt_devres.log
FDA_VERBOSE=2 timeout 600 python tools/build_times.py --configs 4 5 > gpurun_out/build_times_devres.log 2>&1
grep -v "^\s*$" gpurun_out/build_times_devres.log | tail -40
