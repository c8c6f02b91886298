"""Oracle vs oracle on config 4: perturb the rigid-body candidates that enter
every tentative prolongation by 1e-14 (relative) and compare the first 20 PCG residuals with the committed
tests/golden/config4_history.npz.  Shows how much of the device/oracle
trajectory difference the rank-deficient two-node aggregates produce on their
own (full-size parity item 12).  CPU, ~4 min."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402


def main():
    ref = np.load(os.path.join(ROOT, "tests", "golden", "config4_history.npz"))
    w = P.CONFIGS[4]()
    leg = w.solvers[0]
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    B = O.rigid_body_modes(g, w.bc.fixed_dofs)
    rng = np.random.default_rng(0)
    tentative = O.tentative

    def perturbed(agg, Bk, *a, **kw):  # the hybrid builds the SA candidates on the coarse grid
        return tentative(agg, Bk * (1.0 + 1e-14 * rng.standard_normal(Bk.shape)), *a, **kw)

    O.tentative = perturbed
    sm = O.Smoother("chebyshev", 1.0, leg["degree"], lanczos_steps=leg["lanczos_steps"])
    h = O.build_hybrid(g, K, B, leg["n_geo"], leg["coarse_max_dofs"], sm, leg["n_pre"], leg["n_post"],
                       beta=leg["beta"], isolated=leg.get("isolated", "merge"))
    lm = np.array([lv.smoother.lmax_estimate for lv in h.levels[:-1]])
    u, rec = O.pcg(K, w.bc.load_vector, None, h.apply, rtol=w.rtol, max_iterations=20)
    hist = np.array(rec.residual_history)
    print("sizes equal:", [lv.A.shape[0] for lv in h.levels] == list(ref["sizes"]))
    print("lmax rel", np.abs(lm - ref["lmax"]) / ref["lmax"])
    print("trajectory rel diff", np.array2string(np.abs(hist - ref["hist"]) / ref["hist"], precision=2))


if __name__ == "__main__":
    main()
