"""Tensor-core translation path vs the CUDA-core path and the oracle (small cases)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1403_4747_b200 import FDA
    from fda_inputs import icosphere, config_mesh, CONFIGS, random_density
    import oracle as O
    from oracle import fast
    cases = [("ico4 k=40 leaf16", icosphere(4, 0.5), 40.0, 16), ("config1", config_mesh(1), 10.0, 64)]
    for name, (V, F), k, ml in cases:
        x = random_density(len(F), 5)
        el = O.element_geometry(V, F)
        yo = fast.matvec_rows(el, np.arange(len(F)), x, k, 1j / k)
        for lowrank in (1, 0):
            y0 = FDA(V, F, k, 1j / k, 1e-4, max_leaf=ml, m2l_lowrank=lowrank).matvec(x)
            y1 = FDA(V, F, k, 1j / k, 1e-4, max_leaf=ml, m2l_lowrank=lowrank, tensor_cores=1).matvec(x)
            print(f"{name} lowrank={lowrank}: cuda-core {np.linalg.norm(y0-yo)/np.linalg.norm(yo):.3e} "
                  f"tensor-core {np.linalg.norm(y1-yo)/np.linalg.norm(yo):.3e} "
                  f"tc-vs-cc {np.linalg.norm(y1-y0)/np.linalg.norm(y0):.3e}", flush=True)


if __name__ == "__main__":
    main()
