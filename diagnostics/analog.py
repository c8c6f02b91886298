"""Reduced-size analog of a BASELINE config (same generator, smaller grid):
device path vs CPU oracle, per leg -- separates solver bugs from properties of
the seeded density.

    python tools/analog.py CONFIG NX NY [NZ] [--maxit N]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402


def oracle_hierarchy(w, leg, g, K):
    if leg["smoother"] == "chebyshev":
        sm = O.Smoother("chebyshev", 1.0, leg.get("degree", 2))
    else:
        sm = O.Smoother(leg["smoother"], leg.get("weight", 0.5), safeguard=leg.get("safeguard", 0.0))
    B = O.rigid_body_modes(g, w.bc.fixed_dofs)
    if leg["strategy"] == "gmg":
        return O.build_gmg(g, K, 1, sm, leg["n_pre"], leg["n_post"], max_levels=leg["levels"])
    if leg["strategy"] == "amg":
        return O.build_sa_amg(K, B, leg["coarse_max_dofs"], sm, leg["n_pre"], leg["n_post"], beta=leg["beta"],
                              isolated=leg.get("isolated", "merge"))
    return O.build_hybrid(g, K, B, leg["n_geo"], leg["coarse_max_dofs"], sm, leg["n_pre"], leg["n_post"],
                          beta=leg["beta"], isolated=leg.get("isolated", "merge"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("dims", type=int, nargs="+")
    ap.add_argument("--maxit", type=int, default=3000)
    ap.add_argument("--no-gpu", action="store_true")
    a = ap.parse_args()
    w = P.CONFIGS[a.config](dims=tuple(a.dims))
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    f = w.bc.load_vector
    for leg in w.solvers:
        t = time.time()
        ho = oracle_hierarchy(w, leg, g, K)
        uo, reco = O.pcg(K, f, None, ho.apply, rtol=w.rtol, max_iterations=a.maxit)
        line = "%s dofs %d oracle: levels %s iters %d conv %s true-res %.2e C %.10e (%.0fs)" % (
            P.leg_name(leg), g.n_dofs, [lv.A.shape[0] for lv in ho.levels], reco.iterations, reco.converged,
            np.linalg.norm(f - K @ uo) / np.linalg.norm(f), f @ uo, time.time() - t)
        if not a.no_gpu:
            import paper_2001_01655_b200 as T
            from bench import LegRunner
            Kd = T.assemble_stiffness(w.mesh, w.bc, E)
            h = LegRunner(w, leg).build(Kd)
            u, rec = T.cg_solve(Kd, f, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=a.maxit))
            u = u.cpu().numpy()
            x = np.random.default_rng(0).standard_normal(g.n_dofs)
            vc = np.linalg.norm(h.apply(x).cpu().numpy() - ho.apply(x)) / np.linalg.norm(ho.apply(x))
            line += " | gpu: levels %s iters %d conv %s vcycle-rel %.1e u-rel %.1e C %.10e" % (
                [lv.size for lv in h.levels], rec.iterations, rec.converged, vc,
                np.linalg.norm(u - uo) / np.linalg.norm(uo), f @ u)
        print(line, flush=True)


if __name__ == "__main__":
    main()
