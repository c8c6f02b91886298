"""Per-kernel HBM roofline table of one BASELINE config (graph-timed phases).

    python tools/roofline_table.py --config 1 [--legs gmg,amg]

For every level of every leg: the smoother sweep, the residual, the restriction
and the prolongation (and the coarsest solve), each timed as one replay of a
CUDA graph of 50 back-to-back launches (tmg_hierarchy_time_smoother / _phase),
next to its ALGORITHMIC bytes per launch (each array the kernel must touch,
read or written once) -> achieved GB/s and the fraction of the measured HBM
copy bandwidth (MEASURED_PEAKS.json).  Working sets below the 126 MB L2 can
exceed 1.0: they are L2-, not HBM-resident between launches.
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

F8 = 8
def _fp64_peak():
    """Measured DFMA peak of the pool's B200 (tools/fp64_peak.cu -> profiles/r02_fp64_peak.json)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")))["fp64_dfma_tflops"])
    except Exception:  # noqa: BLE001
        return 34.2


FP64_PEAK_TF = _fp64_peak()
# FP64 pipe instructions per element of the character-basis Hex8 operator
# (tmg_fine3h.cuh): 24 face-transform adds, 24 z-combinations, 45 KE^ terms, 42
# accumulations, 24 inverse-transform adds, 6 neighbour adds (+ ~10 epilogue);
# each occupies one issue slot of the FP64 pipe whether it is an add or an FMA,
# so the pipe fraction is instructions / (peak FMA rate)
F3H_DP_PER_ELEMENT = 175.0


def level_bytes(h, k, ndim, mesh, n_levels, cheb=False):
    """(sweep, residual, restrict, prolong) algorithmic bytes of level k.  cheb: the
    timed sweep is one Chebyshev step (r, D^-1, p, x in; x, p', r' out)."""
    lv = h.levels[k]
    n = lv.size
    nxt = h.levels[k + 1].size if k + 1 < n_levels else 0
    if lv.storage == "matrix_free":
        nodes, nel = mesh.node_count, mesh.element_count
        op = nel * F8 + nodes  # moduli + free-dof masks
    elif lv.storage == "stencil":
        op = lv.nonzeros * F8
    else:
        dims = (C.c_int64 * 4)()
        from paper_2001_01655_b200 import _lib
        _lib.check(_lib.load().tmg_hierarchy_export(h.handle, k, 0, dims, None, None, None, None))
        nnzb = int(dims[2])
        op = lv.nonzeros * F8 + nnzb * 4 + (int(dims[0]) + 1) * 4
    sweep = op + (7 if cheb else 4) * n * F8  # Jacobi: x, b, D^-1 in; x' out.  Chebyshev step: 4 in, 3 out
    resid = op + 3 * n * F8  # x, b in; r out
    if lv.provenance == "geometric" or k + 1 >= n_levels:
        restrict = n * F8 + 3 * nxt * F8  # r in; b_c, x_c out, D_c^-1 in
        prolong = nxt * F8 + 2 * n * F8   # e in; x in/out
    else:
        dims = (C.c_int64 * 4)()
        from paper_2001_01655_b200 import _lib
        _lib.check(_lib.load().tmg_hierarchy_export(h.handle, k, 1, dims, None, None, None, None))
        nnzb, rc = int(dims[2]), int(dims[3])
        pbytes = nnzb * ((rc // 1000) * (rc % 1000) * F8 + 4)
        restrict = pbytes + (nxt + 1) * 4 + n * F8 + 3 * nxt * F8
        prolong = pbytes + (n // ((rc // 1000) or 1) + 1) * 4 + nxt * F8 + 2 * n * F8
    return sweep, resid, restrict, prolong


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--legs", default="")
    p.add_argument("--reps", type=int, default=50)
    a = p.parse_args()
    import torch

    import paper_2001_01655_b200 as T
    from bench import LegRunner
    from paper_2001_01655_b200 import _lib, problems
    L = _lib.load()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    w = problems.CONFIGS[a.config]()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    E = law.modulus(torch.as_tensor(w.rho, device="cuda"))
    K = T.StiffnessOperator(w.mesh, w.bc, E)
    print("# config %d (%s), %d dofs; peak %.0f GB/s (MEASURED_PEAKS.json hbm_gbs)" % (a.config, w.name, w.ndof, peak))
    print("# %-6s %-3s %-11s %9s  %-9s %10s %8s %9s %6s" % ("leg", "lvl", "storage", "dofs", "phase", "bytes",
                                                          "us", "GB/s", "frac"))
    ms = C.c_double()
    rows = []
    for leg in w.solvers:
        if a.legs and leg["strategy"] not in a.legs.split(","):
            continue
        lr = LegRunner(w, leg)
        h = lr.build(K)
        nl = h.n_levels
        for k in range(nl):
            lv = h.levels[k]
            if k == nl - 1:
                _lib.check(L.tmg_hierarchy_time_phase(h.handle, k, 3, a.reps, C.byref(ms), None))
                phases = [("coarse", lv.size * lv.size * F8 if k > 0 else 0, ms.value)]
            else:
                b = level_bytes(h, k, w.mesh.ndim, w.mesh, nl, cheb=leg["smoother"] == "chebyshev")
                phases = []
                _lib.check(L.tmg_hierarchy_time_smoother(h.handle, k, a.reps, C.byref(ms), None))
                phases.append(("sweep", b[0], ms.value))
                for ph, nm, by in ((0, "residual", b[1]), (1, "restrict", b[2]), (2, "prolong", b[3])):
                    _lib.check(L.tmg_hierarchy_time_phase(h.handle, k, ph, a.reps, C.byref(ms), None))
                    phases.append((nm, by, ms.value))
            for nm, by, t in phases:
                gbs = by / (t * 1e-3) / 1e9 if t > 0 else 0.0
                row = dict(leg=lr.name, level=k, storage=lv.storage, dofs=lv.size, phase=nm, bytes=by,
                           us=t * 1e3, gbs=gbs, frac=gbs / peak)
                extra = ""
                if lv.storage == "matrix_free" and w.mesh.ndim == 3 and nm in ("sweep", "residual"):
                    # FP64-pipe occupancy of the Hex8 operator: DP instructions per
                    # second against the measured DFMA issue rate (peak TF/s / 2)
                    gi = F3H_DP_PER_ELEMENT * w.mesh.element_count / (t * 1e-3) / 1e12
                    row.update(fp64_tinstr=gi, fp64_frac=gi / (FP64_PEAK_TF / 2))
                    extra = "   FP64 pipe %.2f T instr/s = %.2f of the measured %.1f (= %.1f TF/s / 2)" % (
                        gi, gi / (FP64_PEAK_TF / 2), FP64_PEAK_TF / 2, FP64_PEAK_TF)
                rows.append(row)
                print("  %-6s %3d %-11s %9d  %-9s %10d %8.2f %9.0f %6.2f%s" % (lr.name, k, lv.storage, lv.size, nm, by,
                                                                             t * 1e3, gbs, gbs / peak, extra),
                      flush=True)
    json.dump(rows, open(os.path.join(ROOT, "gpurun_out", "roofline_c%d.json" % a.config), "w"), indent=1)


if __name__ == "__main__":
    main()
