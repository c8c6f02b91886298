"""Every BASELINE config's MG-PCG solve on one GPU: setup, iterations, solve
time, DOF*iterations/s, compliance and the sensitivity kernel (the north-star
per-config report; the bench line measures config 1 only).

    python tools/config_table.py [--configs 0,1,2,3,4] [--maxit 3000]
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="0,1,2,3,4")
    p.add_argument("--maxit", type=int, default=3000)
    a = p.parse_args()
    import torch

    import paper_2001_01655_b200 as T
    from bench import LegRunner
    from paper_2001_01655_b200 import _lib, problems
    from paper_2001_01655_b200._dev import as_dev, empty_dev, ptr, stream_ptr
    L = _lib.load()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    print("# %-34s %-11s %9s %6s %9s %6s %5s %10s %9s %12s %9s %14s" % (
        "workload", "leg", "dofs", "levels", "setup_ms", "iters", "conv", "rel_res", "solve_ms", "DOF*it/s",
        "sens_us", "compliance"))
    for c in [int(x) for x in a.configs.split(",")]:
        w = problems.CONFIGS[c]()
        rho = as_dev(w.rho)
        loads = [w.bc.load_vector] + list(getattr(w, "loads", []) or [])
        for leg in w.solvers:
            lr = LegRunner(w, leg)
            maxit = min(leg.get("max_iterations", a.maxit), a.maxit)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            E = law.modulus(rho)
            K = T.StiffnessOperator(w.mesh, w.bc, E)
            h = lr.build(K)
            torch.cuda.synchronize()
            setup_ms = 1e3 * (time.perf_counter() - t0)
            for li, f in enumerate(loads):
                f_d = as_dev(f)
                u, rec = T.cg_solve(K, f_d, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=maxit))
                dc = empty_dev(w.mesh.element_count)
                comp = C.c_double()
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                _lib.check(L.tmg_compliance_sensitivity(K.handle, ptr(rho), ptr(f_d), ptr(u), law.penalty, law.e_max,
                                                        law.e_min, ptr(dc), C.byref(comp), stream_ptr(None)))
                torch.cuda.synchronize()
                sens_us = 1e6 * (time.perf_counter() - t1)
                hist = rec.residual_history
                name = w.name + ("" if len(loads) == 1 else " load%d" % li)
                print("  %-34s %-11s %9d %6d %9.1f %6d %5s %10.2e %9.2f %12.3e %9.1f %14.6e" % (
                    name, lr.name, w.ndof, h.n_levels, setup_ms if li == 0 else 0.0, rec.iterations,
                    "yes" if rec.converged else "no", hist[-1] / hist[0], 1e3 * rec.solve_time,
                    w.ndof * rec.iterations / max(rec.solve_time, 1e-12), sens_us, comp.value), flush=True)


if __name__ == "__main__":
    main()
