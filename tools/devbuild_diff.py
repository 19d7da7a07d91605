"""Per-kind worst difference between the host and the device build tables (debug)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fda_inputs import icosphere
from paper_1403_4747_b200 import FDA
V, F = icosphere(4, 0.5)
k = 40.0
kw = dict(max_leaf=16, rhs_operator=1)
fh = FDA(V, F, k, -1j / k, 1e-4, build_on_device=0, **kw)
fd = FDA(V, F, k, -1j / k, 1e-4, build_on_device=1, **kw)
mh = fh.table("mats").reshape(-1, 3)
sp = fh.table("specs").reshape(-1, 8)
ph, pd = fh.table("pool"), fd.table("pool")
lr = fh.table("m2l_lr").reshape(-1, 6)
factors = set(lr[:, 3].tolist()) | set(lr[:, 4].tolist())
worst = {}
for i, (off, r, c) in enumerate(mh):
    if i in factors or r * c == 0:
        continue
    a, b = ph[off:off + r * c], pd[off:off + r * c]
    e = float(np.abs(a - b).max() / max(np.abs(a).max(), 1e-30))
    key = (int(sp[i, 0]), int(sp[i, 1]), int(sp[i, 3] >= 0))
    if e > worst.get(key, (0, 0))[0]:
        worst[key] = (e, i)
for key in sorted(worst):
    e, i = worst[key]
    off, r, c = mh[i]
    print("kind,level,dir>=0", key, "worst", f"{e:.2e}", "id", i, "shape", r, c, "spec", sp[i].tolist(),
          "host", ph[off:off + 3], "dev", pd[off:off + 3])
