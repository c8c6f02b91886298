"""Is the Chebyshev smoother's upper bound 1.1 * lambda_hat (10 Lanczos steps)
above the true lambda_max(D^-1 A) on every level of a config's hierarchy?
(CPU, oracle; config 4 takes ~10 min.)

    python diagnostics/lanczos_vs_eigsh.py [--config 4]

A bound below lambda_max would make the Chebyshev polynomial amplify the top of
the spectrum (a divergent smoother, an indefinite V-cycle).  Writes
profiles/r02_lanczos_vs_eigsh_c<config>.txt."""
import argparse
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
import make_checkpoints as MC  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    c = a.config
    w = P.CONFIGS[c]()
    g = O.make_grid(w.mesh.dims)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN))
    lines = ["# config %d: per level, lambda_hat (10 Lanczos steps, the smoother's estimate), the Chebyshev interval's "
             "upper end 1.1 lambda_hat, and lambda_max(D^-1 A) by ARPACK (eigsh on D^-1/2 A D^-1/2, tol 1e-6)" % c,
             "# leg level dofs lambda_hat upper=1.1*lambda_hat lambda_max(eigsh) upper/lambda_max"]
    for leg in w.solvers:
        if leg["smoother"] != "chebyshev":
            continue
        h = MC._build(c, w, g, K, leg, False)
        for k, lv in enumerate(h.levels[:-1]):
            A = sp.csr_matrix(lv.A)
            ds = 1.0 / np.sqrt(A.diagonal())
            S = sp.diags(ds) @ A @ sp.diags(ds)
            t0 = time.time()
            lam = float(spla.eigsh(S, k=1, which="LA", tol=1e-6, return_eigenvectors=False)[0])
            lh = float(lv.smoother.lmax_estimate)
            lines.append("  %-12s %d %9d  %.6f  %.6f  %.6f  %.4f   (%.0f s)" % (
                MC.leg_tag(leg), k, A.shape[0], lh, 1.1 * lh, lam, 1.1 * lh / lam, time.time() - t0))
            print(lines[-1], flush=True)
    out = os.path.join(ROOT, "profiles", "r02_lanczos_vs_eigsh_c%d.txt" % c)
    open(out, "w").write("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
