"""Oracle PCG trajectories on the FULL config-1 workload (BASELINE.json configs[1],
the bench workload): both legs, 2000 iterations, as the bench runs them.

    python tests/golden/make_config1_history.py     (CPU, ~10 min; build container)

Writes tests/golden/config1_history.npz (residual histories + compliance of the
final iterate).  tests/test_gpu_configs.py checks the device trajectories against
it: the early iterations agree to rounding, and neither implementation
converges to rtol 1e-8 within the cap (DESIGN.md deviation 7)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config1_history.npz")


def main():
    w = P.CONFIGS[1]()
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    f = w.bc.load_vector
    out = {}
    for leg in w.solvers:
        t0 = time.time()
        maxit = leg.get("max_iterations", 2000)
        if leg["strategy"] == "gmg":
            sm = O.Smoother(leg["smoother"], leg["weight"], safeguard=leg.get("safeguard", 0.0))
            h = O.build_gmg(g, K, 1, sm, leg["n_pre"], leg["n_post"], max_levels=leg["levels"])
            tag = "gmg"
        else:
            sm = O.Smoother(leg["smoother"], leg["weight"])
            h = O.build_sa_amg(K, O.rigid_body_modes(g, w.bc.fixed_dofs), leg["coarse_max_dofs"], sm, leg["n_pre"],
                               leg["n_post"], beta=leg["beta"], isolated=leg.get("isolated", "merge"))
            tag = "amg"
        t1 = time.time()
        u, rec = O.pcg(K, f, None, h.apply, rtol=w.rtol, max_iterations=maxit)
        out[tag + "_hist"] = np.array(rec.residual_history)
        out[tag + "_sizes"] = np.array([lv.A.shape[0] for lv in h.levels])
        out[tag + "_compliance"] = np.array(f @ u)
        print(tag, "setup %.1f s, %d iterations in %.1f s, rel res %.3e, compliance %.6e" % (
            t1 - t0, rec.iterations, time.time() - t1, rec.residual_history[-1] / rec.residual_history[0], f @ u),
            flush=True)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
