"""Where does the device's config-1 GMG PCG leave the oracle's?  (GPU diagnostic.)

Compares, on the full config (default 1, GMG leg): V-cycles started at each
level, the coarsest solve, and 10-iteration PCG runs of (a) the device,
(b) the oracle, (c) the oracle's PCG loop preconditioned by the DEVICE V-cycle."""
import os
import sys

import numpy as np
import scipy.sparse.linalg as spla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
import paper_2001_01655_b200 as T  # noqa: E402
from bench import LegRunner  # noqa: E402
import make_checkpoints as MC  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
li = int(sys.argv[2]) if len(sys.argv) > 2 else 0
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


print("sizes", [lv.size for lv in h.levels], [lv.A.shape[0] for lv in ho.levels])
print("oracle weights", [getattr(lv.smoother, "w", None) for lv in ho.levels])
print("oracle lmax", [getattr(lv.smoother, "lmax_estimate", None) for lv in ho.levels])
try:
    print("device lmax", [h.level_lmax(k) for k in range(h.n_levels - 1)])
except Exception as e:  # noqa: BLE001
    print("device lmax n/a", e)
for k in range(len(ho.levels) - 1, -1, -1):
    n = ho.levels[k].A.shape[0]
    b = np.random.default_rng(k).standard_normal(n)
    d = h.vcycle(b, k).cpu().numpy()
    o = ho.vcycle(b, k)
    print("level %d: vcycle(random) rel diff %.3e" % (k, rel(d, o)))
d = h.apply(f).cpu().numpy()
o = ho.apply(f)
print("M f: rel diff %.3e" % rel(d, o))
kc = len(ho.levels) - 1
if ho.levels[kc].A.shape[0] < 6000:
    Ac = ho.levels[kc].A.toarray()
    Ad = h.level_matrix(kc).toarray()
    b = np.random.default_rng(5).standard_normal(Ac.shape[0])
    y = h.vcycle(b, kc).cpu().numpy()
    print("coarse: |Ad-Ac|/|Ac| %.2e  dev vs solve(Ad) %.2e  dev vs solve(Ac) %.2e  solve(Ad) vs solve(Ac) %.2e  bwd err %.2e" % (
        np.linalg.norm(Ad - Ac) / np.linalg.norm(Ac), rel(y, np.linalg.solve(Ad, b)), rel(y, np.linalg.solve(Ac, b)),
        rel(np.linalg.solve(Ad, b), np.linalg.solve(Ac, b)),
        np.linalg.norm(Ad @ y - b) / (np.linalg.norm(Ad, 2) * np.linalg.norm(y))))
for it in (1, 2, 3, 5, 10):
    u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(method="cg", rtol=w.rtol, max_iterations=it))
    xo, reco = O.pcg(Kref, f, None, ho.apply, rtol=w.rtol, max_iterations=it)
    xm, recm = O.pcg(Kref, f, None, lambda r: h.apply(r).cpu().numpy(), rtol=w.rtol, max_iterations=it)
    ud = u.cpu().numpy()
    print("it %2d: device vs oracle %.3e   oracle-loop+device-M vs oracle %.3e   device vs oracle-loop+device-M %.3e   res dev %.4e orc %.4e mix %.4e" % (
        it, rel(ud, xo), rel(xm, xo), rel(ud, xm), rec.residual_history[-1], reco.residual_history[-1],
        recm.residual_history[-1]))
