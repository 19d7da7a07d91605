#!/bin/bash
# Correction pair search: class grids (library) vs the single grid (reference), configs 2-5 meshes.
#   bash tools/pairs/run.sh [configs...]   (libfda.so built; writes one JSON line per config)
set -e
cd "$(dirname "$0")"
g++ -O2 -fopenmp -std=c++17 pairs_check.cpp -L../../paper_1403_4747_b200 -Wl,-rpath,$PWD/../../paper_1403_4747_b200 -lfda -o /tmp/pairs_check
for c in ${@:-2 3 4}; do
  python - "$c" << 'PY'
import sys, numpy as np
sys.path.insert(0, "../..")
from fda_inputs import config_mesh
V, F = config_mesh(int(sys.argv[1]))
with open("/tmp/pairs_mesh.bin", "wb") as f:
    np.array([len(V), len(F)], np.int64).tofile(f)
    np.ascontiguousarray(V, np.float64).tofile(f)
    np.ascontiguousarray(F, np.int32).tofile(f)
PY
  echo -n "{\"config\": $c, \"cores\": $(nproc), \"result\": "; /tmp/pairs_check /tmp/pairs_mesh.bin; echo "}"
done
