"""Device SOR triangular solve vs scipy's spsolve_triangular (the reference's
SOR sweep, multigrid.py:105) on the levels of a BASELINE config's GMG hierarchy.

    python tools/sor_timing.py --config 1
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--levels", type=int, default=5)
    a = p.parse_args()
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    import torch

    import paper_2001_01655_b200 as T
    from paper_2001_01655_b200 import _lib, problems
    L = _lib.load()
    w = problems.CONFIGS[a.config]()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    E = law.modulus(torch.as_tensor(w.rho, device="cuda"))
    K = T.StiffnessOperator(w.mesh, w.bc, E)
    ms = C.c_double()
    for kind in ("sor_chebyshev", "sor_gmres"):
        t0 = time.perf_counter()
        h = T.build_gmg(w.mesh, K, 1, T.SmootherConfig(kind=kind), 2, 2, max_levels=a.levels)
        torch.cuda.synchronize()
        print("%s: build %.1f ms" % (kind, 1e3 * (time.perf_counter() - t0)))
        for k in range(h.n_levels - 1):
            _lib.check(L.tmg_hierarchy_time_smoother(h.handle, k, 20, C.byref(ms), None))
            line = "  level %d (%8d dofs): device SOR solve %9.1f us" % (k, h.levels[k].size, 1e3 * ms.value)
            if kind == "sor_gmres":
                A = h.level_matrix(k)
                Lo = sp.tril(A, format="csr")
                v = np.random.default_rng(0).standard_normal(A.shape[0])
                t0 = time.perf_counter()
                spla.spsolve_triangular(Lo, v, lower=True)
                line += "   scipy spsolve_triangular %9.1f us" % (1e6 * (time.perf_counter() - t0))
            print(line, flush=True)
        _lib.check(L.tmg_hierarchy_time_vcycle(h.handle, 0, 5, C.byref(ms), None))
        print("  V-cycle (2/2): %.1f us" % (1e3 * ms.value), flush=True)


if __name__ == "__main__":
    main()
