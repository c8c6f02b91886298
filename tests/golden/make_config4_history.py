"""Oracle PCG trajectory on the FULL config-4 workload (BASELINE.json configs[4]:
193x97x97 Hex8 nodes, 5,447,811 dofs, hybrid: 3 geometric levels with
Jacobi-Chebyshev, then SA-AMG on the 24x12x12 operator), first 20 iterations.

    python tests/golden/make_config4_history.py     (CPU, ~20-40 min, ~40 GB; build container)

Writes tests/golden/config4_history.npz: level sizes, the Lanczos bounds of the
smoothed levels and the residual history; tests/test_gpu_configs.py compares."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config4_history.npz")


def main():
    t0 = time.time()
    w = P.CONFIGS[4]()
    leg = w.solvers[0]
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    print("assembly %.1f s" % (time.time() - t0), flush=True)
    sm = O.Smoother("chebyshev", 1.0, leg["degree"], lanczos_steps=leg["lanczos_steps"])
    h = O.build_hybrid(g, K, O.rigid_body_modes(g, w.bc.fixed_dofs), leg["n_geo"], leg["coarse_max_dofs"], sm,
                       leg["n_pre"], leg["n_post"], beta=leg["beta"], isolated=leg.get("isolated", "merge"))
    print("setup %.1f s, levels %s" % (time.time() - t0, [lv.A.shape[0] for lv in h.levels]), flush=True)
    t1 = time.time()
    u, rec = O.pcg(K, w.bc.load_vector, None, h.apply, rtol=w.rtol, max_iterations=20)
    print("20 iterations in %.1f s" % (time.time() - t1), flush=True)
    np.savez_compressed(OUT, sizes=np.array([lv.A.shape[0] for lv in h.levels]),
                        lmax=np.array([lv.smoother.lmax_estimate for lv in h.levels[:-1]]),
                        hist=np.array(rec.residual_history))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
