import sys, numpy as np, torch
sys.path.insert(0, '.')
from fda_inputs import icosphere, random_density
from paper_1403_4747_b200 import FDA
V, F = icosphere(4, 0.5)
f = FDA(V, F, 10.0, 0.1j, 1e-4, device=0)
f.set_profiling(True)
x = torch.from_numpy(random_density(len(F), 1).astype(np.complex64)).cuda()
y = f.matvec(x); torch.cuda.synchronize(); print("ok", y.abs().sum().item())
