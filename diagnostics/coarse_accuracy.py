"""Accuracy of the device's coarsest solve (explicit inverse applied by GEMV)
against numpy on the device's own coarsest matrix: forward and backward error,
for the SA case of test_amg_pcg_matches_oracle[(32,16)] and config 1's GMG leg.
Run with TMG_COARSE=chol|gj.  (GPU diagnostic.)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2001_01655_b200 as T  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
from oracle import topomg_oracle as O  # noqa: E402
from bench import LegRunner  # noqa: E402


def report(name, h):
    kc = h.n_levels - 1
    Ad = h.level_matrix(kc).toarray()
    n = Ad.shape[0]
    rng = np.random.default_rng(5)
    worst_f = worst_b = 0.0
    for _ in range(4):
        b = rng.standard_normal(n)
        y = h.vcycle(b, kc).cpu().numpy()
        ys = np.linalg.solve(Ad, b)
        worst_f = max(worst_f, np.linalg.norm(y - ys) / np.linalg.norm(ys))
        worst_b = max(worst_b, np.linalg.norm(Ad @ y - b) / (np.linalg.norm(Ad, 2) * np.linalg.norm(y)))
    print("%s: n %d cond %.2e  forward err vs numpy %.2e  backward err %.2e  (TMG_COARSE=%s)" % (
        name, n, np.linalg.cond(Ad), worst_f, worst_b, os.environ.get("TMG_COARSE", "chol")))


from test_gpu_amg import clamped  # noqa: E402
mesh, g, bc, rho, E, K, Kref = clamped((32, 16), 7)
B = T.rigid_body_modes(mesh, bc.fixed_dofs)
h = T.build_sa_amg(K, B, 60, T.SmootherConfig(weight=0.6), 2, 2, beta=0.08, isolated="merge")
report("sa(32,16)", h)
u, rec = T.cg_solve(K, bc.load_vector, None, h, T.SolveConfig(method="cg", rtol=1e-8, max_iterations=3000))
print("   PCG iterations", rec.iterations, "converged", rec.converged, "last residuals", rec.residual_history[-3:])
for c, li in ((1, 0), (3, 0)):
    w = P.CONFIGS[c]()
    Kc = T.assemble_stiffness(w.mesh, w.bc, O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN))
    report("config %d leg %d" % (c, li), LegRunner(w, w.solvers[li]).build(Kc))
