#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDA_M2L_DBG=1 timeout 300 python tools/profile_matvec.py --config 4 --warmup 1 --steps 1 > gpurun_out/r02r_dbg4.log 2>&1
FDA_M2L_DBG=1 timeout 300 python tools/profile_matvec.py --config 2 --warmup 1 --steps 1 > gpurun_out/r02r_dbg2.log 2>&1
grep -c m2l_bf gpurun_out/r02r_dbg4.log
