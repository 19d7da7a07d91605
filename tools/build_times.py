#!/usr/bin/env python
"""fda_build phase times (opt.verbose) for configs, device or host build, plus one matvec.

    python tools/build_times.py --configs 4 5 [--host]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fda_inputs import config_mesh, CONFIGS, random_density  # noqa: E402
from paper_1403_4747_b200 import FDA  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", type=int, nargs="+", default=[4])
ap.add_argument("--host", action="store_true")
args = ap.parse_args()
for cfg in args.configs:
    c = CONFIGS[cfg]
    V, F = config_mesh(cfg)
    t = time.perf_counter()
    f = FDA(V, F, c.k, c.alpha, c.eps, verbose=int(os.environ.get("FDA_VERBOSE", "1")), build_on_device=0 if args.host else 1)
    dt = time.perf_counter() - t
    x = random_density(len(F), c.x_seed)
    y = f.matvec(x)
    st = f.stats()
    print(json.dumps({"config": cfg, "N": len(F), "build_s": round(dt, 2), "device_build": not args.host,
                      "t_build_s": st["t_build_s"], "table_bytes": st["table_bytes"],
                      "y_norm": float(np.linalg.norm(y))}), flush=True)
    f.close()
