"""Parity at BASELINE.json's full sizes (configs 1-4).

The CPU oracle cannot run thousands of PCG iterations on 0.6-5.4 M DOFs, so the
full-size checks use what the oracle CAN do at that size (assembly, one
Galerkin hierarchy, one V-cycle, the SA level-0 pieces) and size-independent
properties of the preconditioner (linearity, symmetry).  Integer artefacts are
bit-exact; floating ones use the fp64 summation-order tolerances of the other
parity tests.  Iteration-count parity is covered at reduced sizes in
test_gpu_parity / test_gpu_amg (the seeded config densities are so
ill-conditioned that iteration counts are chaotic even oracle vs oracle, see
DESIGN.md "Config 1 is numerically degenerate")."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import topomg_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2001_01655_b200 as T  # noqa: E402
from bench import LegRunner  # noqa: E402
from paper_2001_01655_b200 import problems as P  # noqa: E402
from test_gpu_amg import spdiff  # noqa: E402
from test_gpu_parity import host, rel  # noqa: E402

_CACHE = {}


def workload(c):
    if c not in _CACHE:
        w = P.CONFIGS[c]()
        E = O.simp_modulus(w.rho, P.PENAL, P.E0, P.EMIN)
        _CACHE[c] = (w, E)
    return _CACHE[c]


def oracle_K(c):
    w, E = workload(c)
    key = ("K", c)
    if key not in _CACHE:
        _CACHE[key] = (O.make_grid(w.mesh.dims), O.assemble_stiffness(O.make_grid(w.mesh.dims), w.bc.fixed_dofs, E))
    return _CACHE[key]


@pytest.mark.parametrize("c", [1, 2, 3])
def test_full_size_operator(c):
    w, E = workload(c)
    g, Kref = oracle_K(c)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    x = np.random.default_rng(c).standard_normal(g.n_dofs)
    assert rel(host(K @ x), Kref @ x) <= 1e-13
    assert rel(host(K.diagonal()), Kref.diagonal()) <= 1e-14


def test_full_size_config1_gmg_hierarchy_and_vcycle():
    w, E = workload(1)
    g, Kref = oracle_K(1)
    leg = w.solvers[0]
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    h = LegRunner(w, leg).build(K)
    sm = O.Smoother("weighted_jacobi", leg["weight"], safeguard=leg["safeguard"])
    ho = O.build_gmg(g, Kref, 1, sm, leg["n_pre"], leg["n_post"], max_levels=leg["levels"])
    assert [lv.size for lv in h.levels] == [lv.A.shape[0] for lv in ho.levels]
    x = np.random.default_rng(11).standard_normal(g.n_dofs)
    for k, lv in enumerate(ho.levels):
        xk = x[:lv.A.shape[0]]
        assert rel(host(h.level_apply(k, xk)), lv.A @ xk) <= 1e-12, k
    # The coarsest Galerkin operator of this density has cond ~5e13: the 1e-16
    # summation-order differences between the two Galerkin products are
    # amplified by cond in ANY direct solve.  Check the device solve by its
    # backward error, and the V-cycle against the oracle at cond * (operator
    # difference).
    kc = len(ho.levels) - 1
    Ac = ho.levels[kc].A.toarray()
    Ad = h.level_matrix(kc).toarray()
    cond = np.linalg.cond(Ac)
    dA = np.linalg.norm(Ad - Ac, 2) / np.linalg.norm(Ac, 2)
    bc = np.random.default_rng(5).standard_normal(Ac.shape[0])
    y = host(h.vcycle(bc, kc))
    assert np.linalg.norm(Ad @ y - bc) <= 1e-14 * np.linalg.norm(Ad, 2) * np.linalg.norm(y)
    assert rel(host(h.apply(x)), ho.apply(x)) <= max(1e-9, 100.0 * cond * max(dA, 2.2e-16))


def test_full_size_config1_sa_level0_pieces():
    w, E = workload(1)
    g, Kref = oracle_K(1)
    leg = w.solvers[1]
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    h = LegRunner(w, leg).build(K)
    B = O.rigid_body_modes(g, w.bc.fixed_dofs)
    S = O.strength_graph(Kref, leg["beta"], 2)
    assert (h.strength(0) != S).nnz == 0                      # bit-exact strength graph
    agg, _ = O.aggregate(S, leg["isolated"])
    agg = O.merge_small(agg, S, 2)
    dagg, rho = h.aggregates(0)
    assert np.array_equal(dagg, agg)                          # bit-exact aggregate ids
    Tt, _ = O.tentative(agg, B, 2)
    # Two effects make single T columns implementation-defined, in ANY code:
    # (1) aggregates whose rigid-mode block is rank deficient get a trailing
    #     Householder column of rounding noise (excluded);
    # (2) for straight-line aggregates the rotation column's Householder pivot is
    #     a 1e-14 cancellation residue, so its sign (LAPACK's beta = -sign(alpha)
    #     ||x||) is arbitrary -> the column may come out negated.  A column sign
    #     leaves P P^T, hence the V-cycle, unchanged: compare up to column signs.
    nv = B.shape[1]
    Td = h.tentative(0).tocsc()
    keep = np.setdiff1d(np.arange(Tt.shape[1]), deficient_columns(agg, B, 2))
    assert keep.size >= 0.99 * Tt.shape[1]
    sgn = np.sign(np.asarray(Td.multiply(Tt).sum(axis=0)).ravel())
    sgn[sgn == 0] = 1.0
    Sg = sp.diags(sgn)
    assert np.mean(sgn < 0) <= 0.02
    assert spdiff((Td @ Sg)[:, keep], Tt.tocsc()[:, keep]) <= 1e-12
    Pp, omega = O.smooth_prolongation(Kref, Tt)  # power method from default_rng(0), as the bench leg
    assert abs(4.0 / (3.0 * rho) / omega - 1.0) <= 1e-12
    assert spdiff((h.prolongation(0).tocsc() @ Sg)[:, keep], Pp.tocsc()[:, keep]) <= 1e-12
    A1 = (Pp.T @ Kref @ Pp).tocsr()
    A1d = (Sg @ h.level_matrix(1) @ Sg).tocsr()
    assert spdiff(A1d[keep][:, keep], A1[keep][:, keep]) <= 1e-11
    assert nv == 3


def deficient_columns(agg, B, bs, tol=1e-8):
    """Columns of T that belong to aggregates with a rank-deficient candidate
    block (the Householder columns past the numerical rank)."""
    nv = B.shape[1]
    order = np.argsort(agg, kind="stable")
    na = int(agg.max()) + 1
    cuts = np.searchsorted(agg[order], np.arange(na + 1))
    cols = []
    for a in range(na):
        nodes = order[cuts[a]:cuts[a + 1]]
        dofs = (nodes[:, None] * bs + np.arange(bs)).ravel()
        sv = np.linalg.svd(B[dofs], compute_uv=False)
        r = int(np.sum(sv > tol * sv[0])) if sv[0] > 0 else 0
        cols.extend(a * nv + np.arange(r, nv))
    return np.array(cols, dtype=int)


@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_full_size_preconditioner_is_linear_and_symmetric(c):
    """M = V-cycle: linear (fixed polynomial smoothers, direct coarse solve) and
    symmetric (n_pre = n_post, restriction = P^T) -- what PCG requires."""
    w, E = workload(c)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    for leg in w.solvers:
        h = LegRunner(w, leg).build(K)
        rng = np.random.default_rng(c)
        x, y = rng.standard_normal(K.shape[0]), rng.standard_normal(K.shape[0])
        Mx, My = host(h.apply(x)), host(h.apply(y))
        Mxy = host(h.apply(2.0 * x - 3.0 * y))
        assert rel(Mxy, 2.0 * Mx - 3.0 * My) <= 1e-9, leg["strategy"]
        a, b = float(x @ My), float(y @ Mx)
        # the coarse operators of these densities have cond 1e6..1e12, so the
        # explicit coarse inverse is symmetric only to cond * eps
        assert abs(a - b) <= 1e-6 * np.linalg.norm(x) * np.linalg.norm(My), leg["strategy"]


# ---------------------------------------------------------------------------
# fixed-iteration parity against the oracle's own full-size runs
# (tests/golden/make_checkpoints.py -> tests/golden/config{1,2,3,4}_checkpoints.npz)
# ---------------------------------------------------------------------------
# None of configs 1-4 meets rtol 1e-8 on the TRUE residual in fp64 (oracle and
# device alike; profiles/r02_attainable_accuracy.txt: the fp64 rounding floor
# of the residual of these densities lies above it), so both implementations run
# to the same iteration cap and the solves are compared where they are well
# posed: at fixed iteration counts k, the compliance f.x_k (= the energy-norm
# progress of CG, monotone) and the iterate x_k itself (16 seeded Gaussian
# projections, tests/ckpt_common.py).  Tolerance per checkpoint:
# max(north-star tolerance, 10 x the oracle's own floor), the floor being how
# far the oracle moves from itself under rounding-level changes only (matvec
# summed transposed, dots in the GPU's block order, 3D SA candidates jittered by
# 1e-14) -- measured exactly on the full iterates by make_checkpoints.py.
import ckpt_common as CK  # noqa: E402

CKPT = {}


def checkpoints(c):
    import os
    if c not in CKPT:
        path = os.path.join(os.path.dirname(__file__), "golden", "config%d_checkpoints.npz" % c)
        if not os.path.exists(path):
            pytest.skip("config%d_checkpoints.npz not generated" % c)
        CKPT[c] = dict(np.load(path))
    return CKPT[c]


def leg_key(leg, li):
    return "%s_l%d" % (P.leg_name(leg).replace("+", "_"), li)


def run_checkpoints(c, legs=None):
    ref = checkpoints(c)
    w, E = workload(c)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    loads = [w.bc.load_vector] + list(w.loads)
    report = []
    for leg in w.solvers:
        if legs and leg["strategy"] not in legs:
            continue
        h = LegRunner(w, leg).build(K)
        for li, f in enumerate(loads):
            key = leg_key(leg, li)
            assert [lv.size for lv in h.levels] == list(ref[key + "_sizes"]), key
            ks, cap = ref[key + "_ks"], int(ref[key + "_iterations"])
            for n, k in enumerate(list(ks) + [cap]):
                u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(method="cg", rtol=w.rtol, max_iterations=int(k)))
                uh = host(u)
                final = n == len(ks)
                cr = float(ref[key + "_final_comp"] if final else ref[key + "_comp"][n])
                pr = ref[key + "_final_proj"] if final else ref[key + "_proj"][n]
                fl_c = float(ref[key + "_floor_final_comp"] if final else ref[key + "_floor_comp"][n])
                fl_x = float(ref[key + "_floor_final_x"] if final else ref[key + "_floor_x"][n])
                dc = abs(float(f @ uh) - cr) / abs(cr)
                dx = CK.proj_rel(CK.project(uh), pr)
                report.append((key, int(k), dc, fl_c, dx, fl_x))
                print("%s k=%5d: compliance rel %.2e (oracle floor %.2e)  x rel %.2e (floor %.2e)  iters %d%s" % (
                    key, k, dc, fl_c, dx, fl_x, rec.iterations, "  true res %.2e" % (
                        rec.residual_history[-1] / np.linalg.norm(f))))
                if not final:
                    assert rec.iterations == int(k) and not rec.converged, (key, k, rec.iterations)
                    continue
                # the cap run: the same verdict and iteration count -- unless the TRUE
                # residual sits on its fp64 floor right at rtol (config 2: the
                # oracle's own cap runs end at 1.0e-8 .. 2.4e-7 under rounding-level
                # changes, rtol = 1e-8), where either verdict is a rounding accident
                ref_res = float(ref[key + "_hist"][-1] / ref[key + "_fnorm"])
                dev_res = rec.residual_history[-1] / np.linalg.norm(f)
                same = rec.converged == bool(ref[key + "_converged"]) and rec.iterations == int(ref[key + "_iterations"])
                on_floor = max(ref_res, dev_res) <= 30 * w.rtol and rec.iterations >= 0.95 * int(k)
                assert same or on_floor, (key, rec.iterations, rec.converged, dev_res, ref_res)
    # every checkpoint is evaluated (and printed) before the first failure is raised
    for key, k, dc, fl_c, dx, fl_x in report:
        assert dc <= max(1e-10, 10 * fl_c), (key, k, dc, fl_c)
        assert dx <= max(1e-8, 10 * fl_x), (key, k, dx, fl_x)
    return report


def test_full_size_config1_checkpoints_match_oracle():
    """The bench workload of round 1 (MBB 960x320, GMG-5 and SA-AMG legs on the
    same input), 2000 PCG iterations: x_k and f.x_k at k = 10, 50, 200, 1000,
    2000 against the oracle's run."""
    run_checkpoints(1)


def test_full_size_config2_checkpoints_match_oracle():
    """2.46 M dofs, SA-AMG, the four load cases on one hierarchy: k = 10, 50, 200
    and the 300-iteration cap (the recursive residual meets 1e-8 at ~290, the
    true one stays on its fp64 floor 2e-8..1e-7, so restarts follow)."""
    run_checkpoints(2)


def test_full_size_config3_checkpoints_match_oracle():
    """3D GMG-4, Jacobi-Chebyshev: k = 10 .. 3000 against the oracle's 3000-
    iteration run (its Lanczos bounds to 1e-12)."""
    ref = checkpoints(3)
    w, E = workload(3)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    h = LegRunner(w, w.solvers[0]).build(K)
    lm = np.array([h.level_lmax(k) for k in range(h.n_levels - 1)])
    assert np.max(np.abs(lm - ref["gmg4_l0_lmax"]) / ref["gmg4_l0_lmax"]) <= 1e-12
    run_checkpoints(3)


def test_full_size_config4_checkpoints_match_oracle():
    """The bench workload (3D hybrid, 5.45 M dofs): k = 10, 50, 200.  The first
    SA level's two-node aggregates carry rank-5 rigid-mode blocks whose trailing
    Householder column is rounding noise in ANY implementation, so
    the oracle's own floor here includes 1e-14 jitter of the SA candidates."""
    ref = checkpoints(4)
    w, E = workload(4)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    h = LegRunner(w, w.solvers[0]).build(K)
    lm = np.array([h.level_lmax(k) for k in range(h.n_levels - 1)])
    rl = np.abs(lm - ref["hybrid3_amg_l0_lmax"]) / ref["hybrid3_amg_l0_lmax"]
    assert rl[:4].max() <= 1e-12  # the geometric levels and the first SA level
    run_checkpoints(4)
