"""Reduced config-1 analog (same generator, smaller grid): GPU vs oracle per leg.

    python tools/c1_analog.py NX NY CORR MAXIT
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
import paper_2001_01655_b200 as T  # noqa: E402


def main():
    nx, ny, cl, maxit = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
    legs = sys.argv[5].split(",") if len(sys.argv) > 5 else ["gmg", "amg-drop"]
    import torch
    mesh, bc = P._mbb(nx, ny)
    g = P.gaussian_field((nx, ny), cl, 1655)
    rho = P.to_elements(P.cone_filter(P.threshold(g, 0.4), 1.5))
    gr = O.make_grid((nx, ny))
    E = O.simp_modulus(rho, 3, 1, 1e-9)
    Kref = O.assemble_stiffness(gr, bc.fixed_dofs, E)
    K = T.assemble_stiffness(mesh, bc, E)
    f = bc.load_vector
    B = O.rigid_body_modes(gr, bc.fixed_dofs)
    jac = O.Smoother("weighted_jacobi", 0.6, safeguard=1.8)
    tj = T.SmootherConfig(weight=0.6, safeguard=1.8)
    for leg in legs:
        iso = leg.split("-")[1] if "-" in leg else "merge"
        if leg == "gmg":
            ho = O.build_gmg(gr, Kref, 1, jac, 2, 2, max_levels=5)
            h = T.build_gmg(mesh, K, 1, tj, 2, 2, max_levels=5)
        else:
            ho = O.build_sa_amg(Kref, B, 499, O.Smoother("weighted_jacobi", 0.6), 2, 2, beta=P.BETA, isolated=iso)
            h = T.build_sa_amg(K, B, 499, T.SmootherConfig(weight=0.6), 2, 2, beta=P.BETA, isolated=iso)
        uo, reco = O.pcg(Kref, f, None, ho.apply, rtol=1e-8, max_iterations=maxit)
        u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(rtol=1e-8, max_iterations=maxit))
        u = u.cpu().numpy()
        x = np.random.default_rng(0).standard_normal(gr.n_dofs)
        print(leg, "levels", [lv.A.shape[0] for lv in ho.levels], [lv.size for lv in h.levels],
              "iters oracle %d gpu %d" % (reco.iterations, rec.iterations), reco.converged, rec.converged,
              "vcycle rel %.2e" % (np.linalg.norm(h.apply(x).cpu().numpy() - ho.apply(x)) / np.linalg.norm(ho.apply(x))),
              "u rel %.2e" % (np.linalg.norm(u - uo) / np.linalg.norm(uo)),
              "C %.10e %.10e" % (f @ uo, f @ u), flush=True)


if __name__ == "__main__":
    main()
