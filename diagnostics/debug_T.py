"""Find aggregates whose device tentative block differs from the oracle (config 1 AMG leg)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
import paper_2001_01655_b200 as T  # noqa: E402
from bench import LegRunner  # noqa: E402

w = P.config_1()
E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
g = O.make_grid(w.mesh.dims)
Kref = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
leg = w.solvers[1]
K = T.assemble_stiffness(w.mesh, w.bc, E)
h = LegRunner(w, leg).build(K)
B = O.rigid_body_modes(g, w.bc.fixed_dofs)
S = O.strength_graph(Kref, leg["beta"], 2)
agg, _ = O.aggregate(S, leg["isolated"])
agg = O.merge_small(agg, S, 2)
Tt, _ = O.tentative(agg, B, 2)
Td = h.tentative(0).tocsr()
D = (Td - Tt).tocoo()
big = np.abs(D.data) > 1e-10
rows, cols = D.row[big], D.col[big]
print("differing entries", big.sum(), "columns", np.unique(cols).size, "aggregates", np.unique(cols // 3).size)
for a in np.unique(cols // 3)[:5]:
    nodes = np.nonzero(agg == a)[0]
    dofs = (nodes[:, None] * 2 + np.arange(2)).ravel()
    sv = np.linalg.svd(B[dofs], compute_uv=False)
    print("agg", a, "nodes", nodes.tolist(), "sv", sv)
    print("  oracle T\n", Tt[dofs][:, a * 3:a * 3 + 3].toarray())
    print("  device T\n", Td[dofs][:, a * 3:a * 3 + 3].toarray())
    print("  B\n", B[dofs])
