"""Host/device time split of one bench step (config 1 legs): wall time of each
drop-in call with a synchronisation after it, PCG capped at --iters.

    python tools/step_breakdown.py [--iters 1]
"""
import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--iters", type=int, default=1)
    p.add_argument("--reps", type=int, default=4)
    a = p.parse_args()
    import torch

    import paper_2001_01655_b200 as T
    from bench import LegRunner
    from paper_2001_01655_b200 import _lib, problems
    from paper_2001_01655_b200._dev import as_dev, empty_dev, ptr, stream_ptr
    L = _lib.load()
    w = problems.CONFIGS[1]()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    rho = as_dev(w.rho)
    f = as_dev(w.bc.load_vector)
    runners = [LegRunner(w, leg) for leg in w.solvers]
    for rep in range(a.reps):
        for lr in runners:
            ts = {}
            sync = torch.cuda.synchronize
            sync(); t = time.perf_counter()
            E = law.modulus(rho); sync(); ts["modulus"] = time.perf_counter() - t; t = time.perf_counter()
            K = T.StiffnessOperator(w.mesh, w.bc, E); sync(); ts["operator"] = time.perf_counter() - t
            t = time.perf_counter()
            h = lr.build(K); sync(); ts["build"] = time.perf_counter() - t; t = time.perf_counter()
            u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=a.iters)); sync()
            ts["cg_solve"] = time.perf_counter() - t
            ts["  (device solve)"] = rec.solve_time
            t = time.perf_counter()
            dc = empty_dev(w.mesh.element_count)
            comp = C.c_double()
            _lib.check(L.tmg_compliance_sensitivity(K.handle, ptr(rho), ptr(f), ptr(u), law.penalty, law.e_max,
                                                    law.e_min, ptr(dc), C.byref(comp), stream_ptr(None)))
            sync(); ts["sensitivity"] = time.perf_counter() - t
            t = time.perf_counter()
            del h, K; sync(); ts["teardown"] = time.perf_counter() - t
            if rep == a.reps - 1:
                print(lr.name, "  ".join("%s %.2f ms" % (k, 1e3 * v) for k, v in ts.items()), flush=True)


if __name__ == "__main__":
    main()
