"""Short MG-PCG run of one BASELINE config for ncu (few iterations, one step).

    python tools/profile_case.py --config 1 --iters 20
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--reps", type=int, default=2)
    a = p.parse_args()
    import torch

    import paper_2001_01655_b200 as T
    from paper_2001_01655_b200 import problems
    w = problems.CONFIGS[a.config]()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    for leg in [s for s in w.solvers if s["strategy"] == "gmg"]:
        for _ in range(a.reps):
            E = law.modulus(torch.as_tensor(w.rho, device="cuda"))
            K = T.StiffnessOperator(w.mesh, w.bc, E)
            h = T.build_gmg(w.mesh, K, 1, problems.gmg_settings(leg), leg["n_pre"], leg["n_post"],
                            max_levels=leg["levels"])
            u, rec = T.cg_solve(K, w.bc.load_vector, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=a.iters))
            torch.cuda.synchronize()
            print(leg["strategy"], leg.get("levels"), "iters", rec.iterations, "solve_ms", rec.solve_time * 1e3,
                  "res", rec.residual_history[-1] / rec.residual_history[0], flush=True)


if __name__ == "__main__":
    main()
