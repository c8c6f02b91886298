"""Short MG-PCG run of one BASELINE config (every leg) for timing / ncu.

    python tools/profile_case.py --config 1 --iters 20 [--legs gmg,amg]
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--legs", default="")
    a = p.parse_args()
    import torch

    import paper_2001_01655_b200 as T
    from bench import LegRunner
    from paper_2001_01655_b200 import problems
    w = problems.CONFIGS[a.config]()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    rho = torch.as_tensor(w.rho, device="cuda")
    for leg in w.solvers:
        if a.legs and leg["strategy"] not in a.legs.split(","):
            continue
        lr = LegRunner(w, leg)
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            E = law.modulus(rho)
            K = T.StiffnessOperator(w.mesh, w.bc, E)
            h = lr.build(K)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            u, rec = T.cg_solve(K, w.bc.load_vector, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=a.iters))
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            print(lr.name, "levels", [lv.size for lv in h.levels], "flags", h.flags, "setup_ms %.1f" % (1e3 * (t1 - t0)),
                  "iters", rec.iterations, "solve_ms %.1f" % (1e3 * (t2 - t1)),
                  "res %.3e" % (rec.residual_history[-1] / rec.residual_history[0]), flush=True)


if __name__ == "__main__":
    main()
