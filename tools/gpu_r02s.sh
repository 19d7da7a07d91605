#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDA_VERBOSE=2 timeout 900 python tools/build_times.py --configs 5 > gpurun_out/r02s_build.jsonl 2> gpurun_out/r02s_build.err
timeout 600 python tools/ab_options.py --config 4 --steps 20 --variants '{}' > gpurun_out/r02s_ab4.jsonl 2> gpurun_out/r02s_ab4.err
timeout 600 python tools/ab_options.py --config 2 --steps 20 --variants '{}' > gpurun_out/r02s_ab2.jsonl 2> gpurun_out/r02s_ab2.err
timeout 900 python tools/config5.py --cfg 5 --no-oracle > gpurun_out/r02s_config5.json 2> gpurun_out/r02s_config5.err
