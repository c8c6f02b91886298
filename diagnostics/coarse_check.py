"""Backward error of the coarsest-level direct solve (device explicit inverse vs
scipy splu) on a config analog: separates conditioning from solver error."""
import os
import sys

import numpy as np
import scipy.sparse.linalg as spla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
import paper_2001_01655_b200 as T  # noqa: E402

c, dims = int(sys.argv[1]), tuple(int(a) for a in sys.argv[2:])
w = P.CONFIGS[c](dims=dims) if dims else P.CONFIGS[c]()
E = O.simp_modulus(w.rho, 3, 1, 1e-9)
Kd = T.assemble_stiffness(w.mesh, w.bc, E)
if dims:
    h = T.build_gmg(w.mesh, Kd, 999, T.SmootherConfig(kind="chebyshev", weight=1.0), 1, 1)
else:  # the config's own first leg
    from bench import LegRunner
    h = LegRunner(w, w.solvers[0]).build(Kd)
k = h.n_levels - 1
A = h.level_matrix(k).toarray()
b = np.random.default_rng(0).standard_normal(A.shape[0])
y_gpu = h.vcycle(b, k).cpu().numpy()
y_lu = spla.splu(h.level_matrix(k).tocsc()).solve(b)
y_np = np.linalg.solve(A, b)
be = lambda y: np.linalg.norm(A @ y - b) / (np.linalg.norm(A, 2) * np.linalg.norm(y))
print("cond %.2e | backward err gpu %.2e splu %.2e numpy %.2e | rel diff gpu-splu %.2e numpy-splu %.2e" % (
    np.linalg.cond(A), be(y_gpu), be(y_lu), be(y_np), np.linalg.norm(y_gpu - y_lu) / np.linalg.norm(y_lu),
    np.linalg.norm(y_np - y_lu) / np.linalg.norm(y_lu)))
