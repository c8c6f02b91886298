"""Per-level cost split of one PCG iteration on a BASELINE config (graph replays).

    python tools/iter_breakdown.py --config 1
Prints, per leg: PCG ms/iteration, V-cycle time started at each level, and the
graph-timed smoother sweep of each level.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--iters", type=int, default=300)
    p.add_argument("--legs", default="")
    a = p.parse_args()
    import torch

    import paper_2001_01655_b200 as T
    from bench import LegRunner
    from paper_2001_01655_b200 import _lib, problems
    L = _lib.load()
    w = problems.CONFIGS[a.config]()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    E = law.modulus(torch.as_tensor(w.rho, device="cuda"))
    K = T.StiffnessOperator(w.mesh, w.bc, E)
    f = torch.as_tensor(w.bc.load_vector, device="cuda")
    u, rec = T.cg_solve(K, f, None, None, T.SolveConfig(rtol=1e-12, max_iterations=a.iters))
    print("unpreconditioned CG: %.1f us/iter" % (1e6 * rec.solve_time / max(rec.iterations, 1)))
    for leg in w.solvers:
        if a.legs and leg["strategy"] not in a.legs.split(","):
            continue
        lr = LegRunner(w, leg)
        h = lr.build(K)
        u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(rtol=1e-12, max_iterations=a.iters))
        u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(rtol=1e-12, max_iterations=a.iters))
        print("%s: PCG %.1f us/iter (%d its)" % (lr.name, 1e6 * rec.solve_time / rec.iterations, rec.iterations))
        ms = C.c_double()
        for k in range(h.n_levels):
            _lib.check(L.tmg_hierarchy_time_vcycle(h.handle, k, 50, C.byref(ms), None))
            line = "  level %d (%8d dofs): vcycle-from-here %7.1f us" % (k, h.levels[k].size, 1e3 * ms.value)
            if k < h.n_levels - 1:
                _lib.check(L.tmg_hierarchy_time_smoother(h.handle, k, 50, C.byref(ms), None))
                line += "   sweep %6.2f us" % (1e3 * ms.value)
                for ph, nm in ((0, "resid"), (1, "restrict"), (2, "prolong")):
                    _lib.check(L.tmg_hierarchy_time_phase(h.handle, k, ph, 50, C.byref(ms), None))
                    line += "  %s %6.2f" % (nm, 1e3 * ms.value)
            else:
                _lib.check(L.tmg_hierarchy_time_phase(h.handle, k, 3, 50, C.byref(ms), None))
                line += "   coarse solve %6.2f us" % (1e3 * ms.value)
            print(line, flush=True)


if __name__ == "__main__":
    main()
