"""Config-1 GMG: is the device-vs-oracle gap the conditioning of the coarsest
Galerkin operator (cond 4.6e13) acting on the 5e-15 rounding difference of the
two Galerkin products?  (GPU diagnostic.)"""
import os
import sys

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
import paper_2001_01655_b200 as T  # noqa: E402
from bench import LegRunner  # noqa: E402
import make_checkpoints as MC  # noqa: E402

c, li = 1, 0
w = P.CONFIGS[c]()
E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
g = O.make_grid(w.mesh.dims)
Kref = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
leg = w.solvers[li]
K = T.assemble_stiffness(w.mesh, w.bc, E)
h = LegRunner(w, leg).build(K)
ho = MC._build(c, w, g, Kref, leg, False)
f = w.bc.load_vector


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


z1 = h.apply(f).cpu().numpy()
u1, rec = T.cg_solve(K, f, None, h, T.SolveConfig(method="cg", rtol=w.rtol, max_iterations=1))
z2 = h.apply(f).cpu().numpy()
zo = ho.apply(f)
x1 = u1.cpu().numpy()
print("h.apply(f) repeatable: %.3e" % rel(z2, z1))
print("device M f vs oracle M f: %.3e" % rel(z1, zo))
print("direction of device x1 vs device M f: %.3e ; vs oracle M f: %.3e" % (
    rel(x1 / np.linalg.norm(x1), z1 / np.linalg.norm(z1)), rel(x1 / np.linalg.norm(x1), zo / np.linalg.norm(zo))))
# the oracle V-cycle with ONLY its coarsest matrix replaced by the device's
kc = len(ho.levels) - 1
Ad = sp.csc_matrix(h.level_matrix(kc))
lu = spla.splu(Ad)
old = ho.coarse_solve
ho.coarse_solve = lambda b: lu.solve(b)
zod = ho.apply(f)
print("oracle M f with the DEVICE's coarsest matrix (SuperLU) vs oracle: %.3e ; vs device: %.3e" % (rel(zod, zo), rel(zod, z1)))
for it in (1, 10):
    xo_d, _ = O.pcg(Kref, f, None, ho.apply, rtol=w.rtol, max_iterations=it)
    ho.coarse_solve = old
    xo, _ = O.pcg(Kref, f, None, ho.apply, rtol=w.rtol, max_iterations=it)
    ho.coarse_solve = lambda b: lu.solve(b)
    u, _ = T.cg_solve(K, f, None, h, T.SolveConfig(method="cg", rtol=w.rtol, max_iterations=it))
    ud = u.cpu().numpy()
    print("it %d: oracle[device coarse matrix] vs oracle %.3e ; device vs oracle[device coarse matrix] %.3e ; device vs oracle %.3e" % (
        it, rel(xo_d, xo), rel(ud, xo_d), rel(ud, xo)))
# a rounding-level perturbation of the ORACLE's own Galerkin chain: P^T (A P) instead of (P^T A) P
