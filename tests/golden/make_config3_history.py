"""Oracle PCG trajectory on the FULL config-3 workload (BASELINE.json configs[3]:
97x49x49 Hex8 nodes, 698,691 dofs, GMG 4 levels, Chebyshev degree 2 on D^-1 K
with a 10-step Lanczos bound), first 200 iterations.

    python tests/golden/make_config3_history.py     (CPU, ~10 min; build container)

Writes tests/golden/config3_history.npz: level sizes, the Lanczos bounds per
level and the residual history; tests/test_gpu_configs.py compares the device."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config3_history.npz")


def main():
    t0 = time.time()
    w = P.CONFIGS[3]()
    leg = w.solvers[0]
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    sm = O.Smoother("chebyshev", 1.0, leg["degree"], lanczos_steps=leg["lanczos_steps"])
    h = O.build_gmg(g, K, 1, sm, leg["n_pre"], leg["n_post"], max_levels=leg["levels"])
    print("setup %.1f s, levels %s" % (time.time() - t0, [lv.A.shape[0] for lv in h.levels]), flush=True)
    t1 = time.time()
    u, rec = O.pcg(K, w.bc.load_vector, None, h.apply, rtol=w.rtol, max_iterations=200)
    print("200 iterations in %.1f s, rel res %.3e" % (time.time() - t1, rec.residual_history[-1] / rec.residual_history[0]))
    np.savez_compressed(OUT, sizes=np.array([lv.A.shape[0] for lv in h.levels]),
                        lmax=np.array([lv.smoother.lmax_estimate for lv in h.levels[:-1]]),
                        hist=np.array(rec.residual_history))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
