"""Localize a V-cycle mismatch: compare device vs oracle V-cycles started at
each level (config workload, GMG leg)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
import paper_2001_01655_b200 as T  # noqa: E402
from bench import LegRunner  # noqa: E402

c = int(sys.argv[1])
w = P.CONFIGS[c]()
E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
g = O.make_grid(w.mesh.dims)
Kref = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
leg = w.solvers[0]
K = T.assemble_stiffness(w.mesh, w.bc, E)
h = LegRunner(w, leg).build(K)
sm = O.Smoother("weighted_jacobi", leg["weight"], safeguard=leg.get("safeguard", 0.0))
ho = O.build_gmg(g, Kref, 1, sm, leg["n_pre"], leg["n_post"], max_levels=leg["levels"])
print("oracle weights", [getattr(lv.smoother, "w", None) for lv in ho.levels])
for k in range(len(ho.levels) - 1, -1, -1):
    n = ho.levels[k].A.shape[0]
    b = np.random.default_rng(k).standard_normal(n)
    d = h.vcycle(b, k).cpu().numpy()
    o = ho.vcycle(b, k)
    print("level %d: vcycle rel diff %.3e  |o| %.3e" % (k, np.linalg.norm(d - o) / np.linalg.norm(o), np.linalg.norm(o)))
