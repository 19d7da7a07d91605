# ncu of the fused tensor-core M2L kernel (opt.lr_tensor_cores=1) on config 2
TAG=${1:-lrtc}
mkdir -p gpurun_out
cat > /tmp/pm.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from fda_inputs import config_mesh, CONFIGS, random_density
from paper_1403_4747_b200 import FDA
c = CONFIGS[2]; V, F = config_mesh(2)
f = FDA(V, F, c.k, c.alpha, c.eps, max_leaf=c.max_leaf, lr_tensor_cores=int(sys.argv[1]))
x = torch.from_numpy(random_density(len(F), c.x_seed).astype(np.complex64)).cuda()
y = torch.empty_like(x)
f.set_profiling(True)
for _ in range(2): f.matvec(x, y)
torch.cuda.synchronize(); print("ok")
PY
timeout 300 python /tmp/pm.py 1 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python /tmp/pm.py 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_m2l_tc -c 4 -o gpurun_out/$TAG python /tmp/pm.py 1 > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"
