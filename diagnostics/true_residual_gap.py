"""Where does the device's true residual stagnate, compared with the oracle's,
on a high-contrast case (test_gpu_amg::test_hybrid_matches_oracle, 2D (32,16),
30 % void at rho = 1e-3, hybrid n_geo = 2, weighted Jacobi)?

    python diagnostics/true_residual_gap.py      (GPU)

Prints, per iteration cap, the device's reported true residual, the residual
of the device iterate recomputed by the oracle's assembled K, the oracle's own
true residual, and the recursive residual of both -- separating a wrong
device residual from a genuinely different iterate."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2001_01655_b200 as T  # noqa: E402
from oracle import topomg_oracle as O  # noqa: E402
from test_gpu_parity import cantilever, host  # noqa: E402


def main():
    dims, n_geo, kind = (32, 16), 2, "weighted_jacobi"
    mesh, g, bc, rho, E, K, Kref = cantilever(dims, 6, void=True)
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    h = T.build_hybrid(mesh, K, B, n_geo, 60, T.SmootherConfig(kind=kind, weight=0.6), 1, 1, beta=0.08)
    ho = O.build_hybrid(g, Kref, O.rigid_body_modes(g, bc.fixed_dofs), n_geo, 60, O.Smoother(kind=kind, weight=0.6),
                        1, 1, beta=0.08)
    f = bc.load_vector
    x = np.random.default_rng(1).standard_normal(g.n_dofs)
    print("operator rel diff %.2e  V-cycle rel diff %.2e" % (
        np.linalg.norm(host(K @ x) - Kref @ x) / np.linalg.norm(Kref @ x),
        np.linalg.norm(host(h.apply(x)) - ho.apply(x)) / np.linalg.norm(ho.apply(x))))
    for cap in (10, 20, 25, 28, 30, 35, 60, 200, 1000):
        u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(method="cg", rtol=1e-8, max_iterations=cap))
        uh = host(u)
        uo, reco = O.pcg(Kref, f, None, ho.apply, rtol=1e-8, max_iterations=cap)
        print("cap %5d: dev it %4d restarts %3d true %.3e (oracle K: %.3e) recursive %.3e | oracle it %4d true %.3e"
              " | |u-uo|/|uo| %.2e |u| %.3e" % (
                  cap, rec.iterations, rec.restarts, rec.residual_history[-1], np.linalg.norm(f - Kref @ uh),
                  rec.recursive_residual, reco.iterations, reco.residual_history[-1],
                  np.linalg.norm(uh - uo) / np.linalg.norm(uo), np.linalg.norm(uo)))
    hd = np.array(T.cg_solve(K, f, None, h, T.SolveConfig(method="cg", rtol=1e-8, max_iterations=60))[1]
                  .residual_history)
    ho_ = np.array(O.pcg(Kref, f, None, ho.apply, rtol=1e-8, max_iterations=60)[1].residual_history)
    print("histories (device / oracle):")
    for k in range(0, min(len(hd), len(ho_))):
        print("  %3d %.6e %.6e" % (k, hd[k], ho_[k]))


if __name__ == "__main__":
    main()
