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


def test_full_size_config2_four_load_cases_share_one_hierarchy():
    w, E = workload(2)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    leg = w.solvers[0]
    h = LegRunner(w, leg).build(K)
    sols = []
    for f in [w.bc.load_vector] + list(w.loads):
        u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=3000))
        assert rec.converged
        r = f - host(K @ u)
        assert np.linalg.norm(r) <= 1e-6 * np.linalg.norm(f)  # true residual (recursive one: 1e-8)
        sols.append(host(u))
    assert all(np.isfinite(u).all() for u in sols)


def test_full_size_config1_pcg_trajectories_match_oracle():
    """The bench workload itself, both legs, 2000 PCG iterations, against the
    oracle's run on the same input (tests/golden/make_config1_history.py): same
    hierarchy sizes, the same early residual trajectory, and the same failure
    mode at the cap (neither reaches rtol 1e-8 on this non-percolating density,
    DESIGN.md deviation 7).  The early agreement is limited by the coarsest
    operators (GMG: 2562 dofs, cond 4.6e13), whose direct solves differ in
    forward error at the percent level between any two implementations
    (device explicit inverse vs scipy splu, tests/diagnostics/coarse_check.py)."""
    import os
    ref = np.load(os.path.join(os.path.dirname(__file__), "golden", "config1_history.npz"))
    w, E = workload(1)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    for leg in w.solvers:
        tag = "gmg" if leg["strategy"] == "gmg" else "amg"
        h = LegRunner(w, leg).build(K)
        assert [lv.size for lv in h.levels] == list(ref[tag + "_sizes"]), tag
        u, rec = T.cg_solve(K, w.bc.load_vector, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=2000))
        hist = np.array(rec.residual_history)
        rh = ref[tag + "_hist"]
        assert len(hist) == len(rh) == 2001, tag
        d = np.abs(hist - rh) / rh
        print(tag, "rel. diff of the first 12 residuals", np.array2string(d[:12], precision=3),
              "final rel. residual gpu %.3e oracle %.3e" % (hist[-1] / hist[0], rh[-1] / rh[0]))
        assert d[:11].max() <= 0.1, (tag, d[:11])
        assert not rec.converged and rh[-1] / rh[0] > w.rtol
        assert 0.1 <= (hist[-1] / hist[0]) / (rh[-1] / rh[0]) <= 10.0, tag


def test_full_size_config2_solves_match_oracle():
    """BASELINE config 2 at full size (2.46 M dofs, SA-AMG, four load cases on one
    hierarchy) against the oracle's own solves (tests/golden/make_config2_reference.py):
    identical hierarchy sizes, converged, iteration counts, compliance and the
    displacement field through 8 seeded random projections and its norm."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "config2_reference.npz")
    if not os.path.exists(path):
        pytest.skip("config2_reference.npz not generated")
    ref = np.load(path)
    w, E = workload(2)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    h = LegRunner(w, w.solvers[0]).build(K)
    assert [lv.size for lv in h.levels] == list(ref["sizes"])
    W = np.random.default_rng(2002).standard_normal((8, w.ndof))
    for li, f in enumerate([w.bc.load_vector] + list(w.loads)):
        u, rec = T.cg_solve(K, f, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=3000))
        uh = host(u)
        it_ref = len(ref["hist%d" % li]) - 1
        c, cr = float(f @ uh), float(ref["compliance%d" % li])
        pr = ref["proj%d" % li]
        print("load %d: iterations gpu %d oracle %d; compliance rel %.2e; |u| rel %.2e; projections rel %.2e" % (
            li, rec.iterations, it_ref, abs(c - cr) / abs(cr),
            abs(np.linalg.norm(uh) - ref["unorm%d" % li]) / ref["unorm%d" % li],
            np.linalg.norm(W @ uh - pr) / np.linalg.norm(pr)))
        # measured: identical iteration counts (291/293/282/289), compliance
        # 6e-12..1.3e-10, projections 7e-9..4e-8 -- both solves stop at rtol 1e-8 on
        # a cond ~1e12 operator, so the 1e-10 / 1e-8 targets sit at the noise floor
        assert rec.converged
        assert abs(rec.iterations - it_ref) <= 1
        assert abs(c - cr) <= 1e-9 * abs(cr)
        assert np.linalg.norm(W @ uh - pr) <= 1e-7 * np.linalg.norm(pr)


def test_full_size_config3_trajectory_matches_oracle():
    """BASELINE config 3 at full size (698,691 dofs, 3D GMG-4, Jacobi-Chebyshev
    degree 2 with Lanczos bounds): the oracle's own first 200 PCG iterations
    (tests/golden/make_config3_history.py) -- same level sizes, same Lanczos
    bounds, the same residual trajectory."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "config3_history.npz")
    if not os.path.exists(path):
        pytest.skip("config3_history.npz not generated")
    ref = np.load(path)
    w, E = workload(3)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    h = LegRunner(w, w.solvers[0]).build(K)
    assert [lv.size for lv in h.levels] == list(ref["sizes"])
    lm = np.array([h.level_lmax(k) for k in range(h.n_levels - 1)])
    u, rec = T.cg_solve(K, w.bc.load_vector, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=200))
    hist, rh = np.array(rec.residual_history), ref["hist"]
    d = np.abs(hist - rh) / rh
    print("lmax rel", np.abs(lm - ref["lmax"]) / ref["lmax"], "trajectory rel diff at 10/50/100/200:",
          [float(d[k]) for k in (10, 50, 100, 200)])
    assert np.max(np.abs(lm - ref["lmax"]) / ref["lmax"]) <= 1e-10
    assert len(hist) == len(rh) == 201
    assert d[:51].max() <= 1e-6  # measured 1e-9 at 10, 1.3e-7 at 50, 2.3e-6 at 200
    assert d.max() <= 1e-5


def test_full_size_config4_trajectory_matches_oracle():
    """BASELINE config 4 at full size (5,447,811 dofs, hybrid: 3 geometric levels
    then SA-AMG, Jacobi-Chebyshev everywhere): the oracle's own first 20 PCG
    iterations (tests/golden/make_config4_history.py) -- same level sizes
    (geometric and aggregated), same Lanczos bounds, same residual trajectory."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "config4_history.npz")
    if not os.path.exists(path):
        pytest.skip("config4_history.npz not generated")
    ref = np.load(path)
    w, E = workload(4)
    K = T.assemble_stiffness(w.mesh, w.bc, E)
    h = LegRunner(w, w.solvers[0]).build(K)
    assert [lv.size for lv in h.levels] == list(ref["sizes"])
    lm = np.array([h.level_lmax(k) for k in range(h.n_levels - 1)])
    u, rec = T.cg_solve(K, w.bc.load_vector, None, h, T.SolveConfig(rtol=w.rtol, max_iterations=20))
    hist, rh = np.array(rec.residual_history), ref["hist"]
    d = np.abs(hist - rh) / rh
    print("lmax rel", np.abs(lm - ref["lmax"]) / ref["lmax"], "trajectory rel diff:", np.array2string(d, precision=2))
    # The first SA level (407 aggregates on the 12,675-dof operator) has 36
    # two-node aggregates: two 3-dof nodes carry a rank-5 block of the 6 rigid
    # modes, so one Householder column of T per such aggregate is rounding noise
    # in ANY implementation (reference included, DESIGN.md "Case excluded on
    # purpose"); the operators below it, their Lanczos bound (8.6e-4) and from
    # iteration 1 the trajectory (0.2-0.5 %, growing to 1-2 % by iteration 20)
    # differ for that reason alone: the oracle against itself with the SA
    # candidates perturbed by 1e-14 shows the same (deepest bound 1.2e-3,
    # trajectory 1-2 %; diagnostics/config4_noise_drift.py).
    rl = np.abs(lm - ref["lmax"]) / ref["lmax"]
    assert rl[:4].max() <= 1e-12  # the geometric levels and the first SA level
    assert len(hist) == len(rh) == 21
    assert d[0] <= 1e-12                  # same load vector, same initial residual
    assert d[:5].max() <= 1e-2
    assert d.max() <= 5e-2
