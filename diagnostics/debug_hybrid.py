import sys, numpy as np, scipy.sparse as sp
import os; _R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, 'tests'))
from oracle import topomg_oracle as O
import paper_2001_01655_b200 as T
from test_gpu_parity import cantilever
def spdiff(A, B):
    D = (sp.csr_matrix(A) - sp.csr_matrix(B)).tocoo()
    return (np.max(np.abs(D.data)) if D.nnz else 0.0) / max(np.max(np.abs(sp.csr_matrix(B).data)), 1e-300)
mesh, g, bc, rho, E, K, Kref = cantilever((16, 8, 8), 6, void=True)
for kind, w, ng in (("chebyshev", 1.0, 2), ("weighted_jacobi", 0.6, 2), ("chebyshev", 1.0, 1)):
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    h = T.build_hybrid(mesh, K, B, ng, 60, T.SmootherConfig(kind=kind, weight=w), 1, 1, beta=0.08)
    ho = O.build_hybrid(g, Kref, O.rigid_body_modes(g, bc.fixed_dofs), ng, 60, O.Smoother(kind=kind, weight=w), 1, 1, beta=0.08)
    print(kind, ng, [lv.size for lv in h.levels], [lv.A.shape[0] for lv in ho.levels])
    for k, lv in enumerate(ho.levels):
        line = "L%d A %.2e" % (k, spdiff(h.level_matrix(k), lv.A))
        if lv.provenance == "algebraic" and lv.P is not None:
            S = h.strength(k); agg, r = h.aggregates(k)
            line += " S %d agg %s T %.2e P %.2e rho %.3e/%.3e" % ((S != lv.strength).nnz, np.array_equal(agg, lv.aggregates),
                spdiff(h.tentative(k), lv.tentative), spdiff(h.prolongation(k), lv.P), r, 4/(3*lv.omega))
        print(line)
