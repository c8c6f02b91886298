"""Convergence study of one BASELINE config: residual history of each leg at a
large iteration cap (and variants of the smoother weight safeguard).

    python tools/converge_study.py --config 1 --iters 30000
"""

import argparse
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--iters", type=int, default=30000)
    p.add_argument("--every", type=int, default=1000)
    p.add_argument("--safeguards", default="")
    a = p.parse_args()
    import torch

    import paper_2001_01655_b200 as T
    from bench import LegRunner
    from paper_2001_01655_b200 import problems
    w = problems.CONFIGS[a.config]()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    E = law.modulus(torch.as_tensor(w.rho, device="cuda"))
    K = T.StiffnessOperator(w.mesh, w.bc, E)
    f = torch.as_tensor(w.bc.load_vector, device="cuda")
    variants = [None] + [float(s) for s in a.safeguards.split(",") if s]
    for leg in w.solvers:
        for sg in variants:
            lr = LegRunner(w, leg)
            if sg is not None:
                lr.sm = dataclasses.replace(lr.sm, safeguard=sg)
            h = lr.build(K)
            u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=a.iters))
            hist = np.array(rec.residual_history) / rec.residual_history[0]
            r = f - K @ u
            true_rel = float(torch.linalg.norm(r) / torch.linalg.norm(f))
            print("%s safeguard=%s iters=%d converged=%s final=%.3e min=%.3e true=%.3e compliance=%.12e"
                  % (lr.name, lr.sm.safeguard, rec.iterations, rec.converged, hist[-1], hist.min(), true_rel,
                     float(torch.dot(f, u))), flush=True)
            print("   ", " ".join("%d:%.2e" % (i, hist[i]) for i in range(0, len(hist), a.every)), flush=True)


if __name__ == "__main__":
    main()
