"""GPU parity of the smoothed-aggregation and hybrid hierarchies against the CPU
oracle.  Integer artefacts (strength graph, aggregate ids, level sizes, flags)
must be bit-exact; floating artefacts (T, rho, P, Galerkin operators, V-cycle)
agree to fp64 summation-order tolerance."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import topomg_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2001_01655_b200 as T  # noqa: E402
from test_gpu_parity import (assert_pcg_parity, cantilever, host, iteration_tolerance, rel,  # noqa: E402
                             reproducibility_floor)


def clamped(dims, seed, void=True):
    """cantilever() with every left-edge dof fixed -> isolated strength-graph nodes."""
    return cantilever(dims, seed, void=void)


def oracle_sa(g, Kref, fixed, bound, beta, sm, n_pre=2, n_post=2, isolated="merge"):
    return O.build_sa_amg(Kref, O.rigid_body_modes(g, fixed), bound, sm, n_pre, n_post, beta=beta,
                          isolated=isolated)


def spdiff(A, B):
    D = (sp.csr_matrix(A) - sp.csr_matrix(B)).tocoo()
    return (np.max(np.abs(D.data)) if D.nnz else 0.0) / max(np.max(np.abs(sp.csr_matrix(B).data)), 1e-300)


@pytest.mark.parametrize("dims,beta,isolated", [((12, 8), 0.08, "merge"), ((24, 12), 0.003, "merge"),
                                                ((6, 4, 4), 0.08, "merge"), ((8, 4, 4), 0.003, "merge"),
                                                ((24, 12), 0.08, "drop"), ((8, 4, 4), 0.0064, "drop")])
def test_sa_setup_pieces(dims, beta, isolated):
    mesh, g, bc, rho, E, K, Kref = clamped(dims, 4)
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    h = T.build_sa_amg(K, B, 40, T.SmootherConfig(weight=0.6), 2, 2, beta=beta, isolated=isolated)
    ho = oracle_sa(g, Kref, bc.fixed_dofs, 40, beta, O.Smoother(weight=0.6), isolated=isolated)
    if isolated == "drop":  # the case must exercise the extension: unaggregated nodes exist
        assert (ho.levels[0].aggregates < 0).any()
    assert [lv.size for lv in h.levels] == [lv.A.shape[0] for lv in ho.levels]
    assert sorted(set(h.flags)) == sorted(set(ho.flags))
    assert all(lv.provenance == "algebraic" for lv in h.levels)
    for k, lv in enumerate(ho.levels[:-1]):
        S = h.strength(k)
        assert (S != lv.strength).nnz == 0, k          # bit-exact strength graph
        agg, rho_k = h.aggregates(k)
        assert np.array_equal(agg, lv.aggregates), k   # bit-exact aggregate ids
        assert spdiff(h.tentative(k), lv.tentative) <= 1e-12
        assert abs(rho_k * 3 / 4 * lv.omega - 1.0) <= 1e-12  # omega = 4 / (3 rho)
        assert spdiff(h.prolongation(k), lv.P) <= 1e-12
        assert spdiff(h.level_matrix(k + 1), ho.levels[k + 1].A) <= 1e-11
    x = np.random.default_rng(1).standard_normal(g.n_dofs)
    for k, lv in enumerate(ho.levels):
        xk = x[:lv.A.shape[0]]
        assert rel(host(h.level_apply(k, xk)), lv.A @ xk) <= 1e-11
    assert rel(host(h.apply(x)), ho.apply(x)) <= 1e-9


def test_sa_forced_pairwise_odd():
    # beta so large that no edge is strong -> forced pairwise aggregation; 5x3 -> 24
    # nodes... use 4x2 (15 nodes, odd) so the merge fallback path runs as well
    mesh, g, bc, rho, E, K, Kref = cantilever((4, 2), 2)
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    h = T.build_sa_amg(K, B, 6, T.SmootherConfig(weight=0.6), 1, 1, beta=1e9)
    ho = oracle_sa(g, Kref, bc.fixed_dofs, 6, 1e9, O.Smoother(weight=0.6), 1, 1)
    assert [lv.size for lv in h.levels] == [lv.A.shape[0] for lv in ho.levels]
    assert "forced_pairwise_aggregation" in h.flags
    for k, lv in enumerate(ho.levels[:-1]):
        assert np.array_equal(h.aggregates(k)[0], lv.aggregates)
    b = np.random.default_rng(2).standard_normal(g.n_dofs)
    assert rel(host(h.apply(b)), ho.apply(b)) <= 1e-9


@pytest.mark.parametrize("dims,beta,isolated", [((32, 16), 0.08, "merge"), ((10, 6, 6), 0.08, "merge"),
                                                ((48, 16), 0.08, "drop"), ((12, 6, 6), 0.0064, "drop")])
def test_amg_pcg_matches_oracle(dims, beta, isolated):
    mesh, g, bc, rho, E, K, Kref = clamped(dims, 7)
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    h = T.build_sa_amg(K, B, 60, T.SmootherConfig(weight=0.6), 2, 2, beta=beta, isolated=isolated)
    ho = oracle_sa(g, Kref, bc.fixed_dofs, 60, beta, O.Smoother(weight=0.6), isolated=isolated)
    u, rec = T.cg_solve(K, bc.load_vector, None, h, T.SolveConfig(rtol=1e-8, max_iterations=3000))
    uo, reco = O.pcg(Kref, bc.load_vector, None, ho.apply, rtol=1e-8, max_iterations=3000)
    assert_pcg_parity(rec, host(u), reco, uo, bc.load_vector,
                      reproducibility_floor(Kref, bc.load_vector, ho.apply, maxit=3000, hierarchy=ho))


# (16,8,8) with n_geo=2 is deliberately absent: its second SA level aggregates two
# 6-dof nodes whose candidate block [R_a; R_b] is rank deficient (exact zeros on
# R's diagonal from the 2-node aggregates above), so the trailing Householder
# columns of T are rounding noise in ANY implementation -- the reference is not
# reproducible there either (diagnostics/debug_hybrid.py shows the level-by-level split).
# (32,16): |u| = 3.6e8 with |f| = 1, so the fp64 floor of the TRUE residual,
# ~eps |K| |u| = 8e-8, sits above rtol 1e-8 (device and oracle both stagnate at
# 3e-8..1e-5 while restarting, diagnostics/true_residual_gap.py): the case
# runs at rtol 1e-6, where both meet the reference's true-residual contract.
@pytest.mark.parametrize("dims,n_geo,kind,rtol", [((16, 8, 8), 1, "weighted_jacobi", 1e-8),
                                                  ((16, 8, 8), 1, "chebyshev", 1e-8),
                                                  ((32, 16), 2, "weighted_jacobi", 1e-6),
                                                  ((24, 12, 12), 2, "chebyshev", 1e-8)])
def test_hybrid_matches_oracle(dims, n_geo, kind, rtol):
    mesh, g, bc, rho, E, K, Kref = cantilever(dims, 6, void=True)
    w = 1.0 if kind == "chebyshev" else 0.6
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    h = T.build_hybrid(mesh, K, B, n_geo, 60, T.SmootherConfig(kind=kind, weight=w), 1, 1, beta=0.08)
    ho = O.build_hybrid(g, Kref, O.rigid_body_modes(g, bc.fixed_dofs), n_geo, 60, O.Smoother(kind=kind, weight=w),
                        1, 1, beta=0.08)
    assert [lv.size for lv in h.levels] == [lv.A.shape[0] for lv in ho.levels]
    assert [lv.provenance for lv in h.levels] == [lv.provenance for lv in ho.levels]
    for k, lv in enumerate(ho.levels):
        assert spdiff(h.level_matrix(k), lv.A) <= 1e-11, k
    b = np.random.default_rng(3).standard_normal(g.n_dofs)
    assert rel(host(h.apply(b)), ho.apply(b)) <= 1e-9
    u, rec = T.cg_solve(K, bc.load_vector, None, h, T.SolveConfig(rtol=rtol, max_iterations=3000))
    uo, reco = O.pcg(Kref, bc.load_vector, None, ho.apply, rtol=rtol, max_iterations=3000)
    assert rec.converged
    assert_pcg_parity(rec, host(u), reco, uo, bc.load_vector,
                      reproducibility_floor(Kref, bc.load_vector, ho.apply, rtol=rtol, maxit=3000, hierarchy=ho))


def test_hybrid_full_geo_equals_gmg_and_zero_is_amg():
    mesh, g, bc, rho, E, K, Kref = cantilever((8, 4), 5)
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    hg = T.build_gmg(mesh, K, 40)
    hh = T.build_hybrid(mesh, K, B, hg.n_levels - 1, 40)
    assert [lv.size for lv in hh.levels] == [lv.size for lv in hg.levels]
    b = np.random.default_rng(0).standard_normal(g.n_dofs)
    assert rel(host(hh.apply(b)), host(hg.apply(b))) <= 1e-12
    ha = T.build_sa_amg(K, B, 40)
    h0 = T.build_hybrid(mesh, K, B, 0, 40)
    assert rel(host(h0.apply(b)), host(ha.apply(b))) <= 0.0 + 1e-15


def test_sa_validates_nullspace_shape():
    mesh, g, bc, rho, E, K, Kref = cantilever((4, 2), 1)
    with pytest.raises(ValueError):
        T.build_sa_amg(K, np.ones(g.n_dofs), 20)
    with pytest.raises(ValueError):
        T.build_sa_amg(K, T.rigid_body_modes(mesh, bc.fixed_dofs), 20, isolated="keep")


# Drop-mode cases avoid 3D aggregates of two 3-dof nodes: their 6x6 rigid-mode block
# has rank 5 (rotation about the joining axis vanishes) -- the rank-deficient
# situation described above test_hybrid_matches_oracle.
def test_hybrid_drop_matches_oracle():
    mesh, g, bc, rho, E, K, Kref = cantilever((64, 32), 6, void=True)
    sm = T.SmootherConfig(kind="chebyshev", weight=1.0)
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    h = T.build_hybrid(mesh, K, B, 1, 60, sm, 1, 1, beta=0.08, isolated="drop")
    ho = O.build_hybrid(g, Kref, O.rigid_body_modes(g, bc.fixed_dofs), 1, 60, O.Smoother(kind="chebyshev"),
                        1, 1, beta=0.08, isolated="drop")
    assert [lv.size for lv in h.levels] == [lv.A.shape[0] for lv in ho.levels]
    for k, lv in enumerate(ho.levels):
        assert spdiff(h.level_matrix(k), lv.A) <= 1e-11, k
    b = np.random.default_rng(3).standard_normal(g.n_dofs)
    assert rel(host(h.apply(b)), ho.apply(b)) <= 1e-9
