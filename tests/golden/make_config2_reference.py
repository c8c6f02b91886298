"""Oracle solve of the FULL config-2 workload (BASELINE.json configs[2]: 2.46 M
dofs, SA-AMG, four load cases sharing one hierarchy), as the bench/config table
runs it on the device.

    python tests/golden/make_config2_reference.py     (CPU, long; build container)

The displacements are too large for a fixture, so it stores per load case the
iteration count, the residual history, the compliance f.u, ||u|| and u
projected on 8 seeded random vectors (a 2.46 M-dof field pinned by 8 numbers);
tests/test_gpu_configs.py compares the device solves against them."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config2_reference.npz")


def projections(n, k=8, seed=2002):
    return np.random.default_rng(seed).standard_normal((k, n))


def main():
    t0 = time.time()
    w = P.CONFIGS[2]()
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    leg = w.solvers[0]
    sm = O.Smoother(leg["smoother"], leg["weight"])
    h = O.build_sa_amg(K, O.rigid_body_modes(g, w.bc.fixed_dofs), leg["coarse_max_dofs"], sm, leg["n_pre"],
                       leg["n_post"], beta=leg["beta"], isolated=leg.get("isolated", "merge"))
    print("setup %.1f s, levels %s" % (time.time() - t0, [lv.A.shape[0] for lv in h.levels]), flush=True)
    W = projections(w.ndof)
    out = {"sizes": np.array([lv.A.shape[0] for lv in h.levels])}
    for li, f in enumerate([w.bc.load_vector] + list(w.loads)):
        t1 = time.time()
        u, rec = O.pcg(K, f, None, h.apply, rtol=w.rtol, max_iterations=3000)
        out["hist%d" % li] = np.array(rec.residual_history)
        out["compliance%d" % li] = np.array(f @ u)
        out["unorm%d" % li] = np.array(np.linalg.norm(u))
        out["proj%d" % li] = W @ u
        print("load %d: %d iterations in %.1f s, converged %s, compliance %.9e" % (
            li, rec.iterations, time.time() - t1, rec.converged, f @ u), flush=True)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, "total %.1f s" % (time.time() - t0))


if __name__ == "__main__":
    main()
