"""Is rtol = 1e-8 on the TRUE residual attainable in fp64 for the BASELINE
configs?  (CPU, build container, after tests/golden/make_checkpoints.py.)

    python tools/attainable_accuracy.py [--configs 1,2,3,4] [--scratch /tmp/tmg_ckpt]

The reference's contract (krylov.py:128-129) is ||f - K u|| <= rtol ||f||
evaluated in fp64.  For every config and leg this computes, from the oracle's
assembled K and its last iterate u (the scratch of make_checkpoints.py):

  norm_bound  eps ||K||_2 ||u|| / ||f||           (normwise bound on the rounding
                                                   error of one fp64 residual;
                                                   ||K||_2 by 40 power steps)
  comp_bound  eps || |K| |u| || / ||f||           (componentwise bound)
  round_rms   eps/(2 sqrt 3) sqrt(sum_ij K_ij^2 u_j^2) / ||f||
              -- the expected residual of u ROUNDED to fp64 (uniform relative
                 rounding errors of the entries): an fp64 vector next to the
                 exact solution has at least about this true residual
  eval_noise  ||fl64(f - K u) - (f - K u)|| / ||f||, the second term in 80-bit
              extended precision (numpy longdouble, row sums by reduceat):
              the measured noise of deciding the test at all
  true_res    the extended-precision true residual of the iterate itself

If round_rms (and eval_noise) exceed rtol, no fp64 iterate of the solution can
be shown to meet rtol = 1e-8: the contract is below fp64's attainable
accuracy for that input, in ANY implementation.  Writes
profiles/r02_attainable_accuracy.{txt,json}."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from oracle import topomg_oracle as O  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402

EPS = np.finfo(float).eps


def row_sums_ld(K, w):
    """sum_j K_ij w_j per row in longdouble (w longdouble)."""
    prod = K.data.astype(np.longdouble) * w[K.indices]
    out = np.zeros(K.shape[0], dtype=np.longdouble)
    nz = np.diff(K.indptr) > 0
    out[nz] = np.add.reduceat(prod, K.indptr[:-1][nz])
    return out


def two_norm(K, iters=40, seed=0):
    v = np.random.default_rng(seed).standard_normal(K.shape[0])
    lam = 0.0
    for _ in range(iters):
        v /= np.linalg.norm(v)
        w = K @ v
        lam = float(np.linalg.norm(w))
        v = w
    return lam


def analyse(K, f, u):
    fn = float(np.linalg.norm(f))
    Kn = two_norm(K)
    un = float(np.linalg.norm(u))
    absK = abs(K)
    comp = float(np.linalg.norm(absK @ np.abs(u)))
    K2 = K.copy()
    K2.data = K2.data ** 2
    rms = float(np.sqrt(np.sum(K2 @ (u * u))))
    r64 = f - K @ u
    rld = f.astype(np.longdouble) - row_sums_ld(K, u.astype(np.longdouble))
    noise = float(np.sqrt(np.sum((r64.astype(np.longdouble) - rld) ** 2)))
    tres = float(np.sqrt(np.sum(rld ** 2)))
    return dict(fnorm=fn, K2=Kn, unorm=un, norm_bound=EPS * Kn * un / fn, comp_bound=EPS * comp / fn,
                round_rms=EPS / (2 * np.sqrt(3.0)) * rms / fn, eval_noise=noise / fn, true_res=tres / fn,
                fp64_true_res=float(np.linalg.norm(r64)) / fn)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--scratch", default=os.environ.get("TMG_CKPT_SCRATCH", "/tmp/tmg_ckpt"))
    a = ap.parse_args()
    import make_checkpoints as MC
    rows = []
    for c in [int(x) for x in a.configs.split(",")]:
        w = P.CONFIGS[c]()
        g = O.make_grid(w.mesh.dims)
        K = O.assemble_stiffness(g, w.bc.fixed_dofs, O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)).tocsr()
        loads = [w.bc.load_vector] + list(w.loads)
        for leg in w.solvers:
            tag = MC.leg_tag(leg)
            for li, f in enumerate(loads):
                path = os.path.join(a.scratch, "c%d_%s_l%d_base_xfinal.npy" % (c, tag, li))
                meta = os.path.join(a.scratch, "c%d_%s_l%d_base.npz" % (c, tag, li))
                if not os.path.exists(path):
                    print("missing", path)
                    continue
                u = np.load(path)
                m = dict(np.load(meta))
                row = dict(config=c, leg=tag, load=li, iterations=int(m["iterations"]),
                           converged=bool(m["converged"]), **analyse(K, f, u))
                rows.append(row)
                print(json.dumps(row), flush=True)
        write(rows)


def write(rows):
    """Merge `rows` into profiles/r02_attainable_accuracy.{json,txt} (rows of other
    configs already there are kept: the configs can be analysed one at a time)."""
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    jpath = os.path.join(ROOT, "profiles", "r02_attainable_accuracy.json")
    old = []
    if os.path.exists(jpath):
        old = json.load(open(jpath))
    new_keys = {(r["config"], r["leg"], r["load"]) for r in rows}
    rows = sorted([r for r in old if (r["config"], r["leg"], r["load"]) not in new_keys] + rows,
                  key=lambda r: (r["config"], r["leg"] != "gmg5", r["leg"], r["load"]))
    with open(jpath, "w") as fh:
        json.dump(rows, fh, indent=1)
    with open(os.path.join(ROOT, "profiles", "r02_attainable_accuracy.txt"), "w") as fh:
        fh.write("# python tools/attainable_accuracy.py  (oracle K, the oracle's last iterate u of each leg;"
                 " all quantities relative to ||f||; rtol = 1e-8)\n")
        fh.write("# %-3s %-12s %4s %6s %5s %10s %10s %10s %10s %10s %10s %10s %10s\n" % (
            "cfg", "leg", "load", "iters", "conv", "|K|_2", "|u|", "norm_bnd", "comp_bnd", "round_rms",
            "eval_noise", "true_res", "vs_rtol"))
        for r in rows:
            fh.write("  %-3d %-12s %4d %6d %5s %10.3e %10.3e %10.3e %10.3e %10.3e %10.3e %10.3e %10s\n" % (
                r["config"], r["leg"], r["load"], r["iterations"], "yes" if r["converged"] else "no", r["K2"],
                r["unorm"], r["norm_bound"], r["comp_bound"], r["round_rms"], r["eval_noise"], r["true_res"],
                "above" if r["round_rms"] > 1e-8 else "below"))
    print("wrote profiles/r02_attainable_accuracy.{txt,json} (%d rows)" % len(rows))


if __name__ == "__main__":
    main()
