"""Pin the CPU oracle against golden vectors produced by the reference itself.

tests/golden/make_golden.py ran /root/reference/pkg/src/topomg on these exact
inputs; every comparison here is oracle-vs-reference.  Integer outputs (strength
graphs, aggregate ids, level sizes) must be bit-exact.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import topomg_oracle as O


def cantilever(dims, seed, void=False):
    """Same inputs as make_golden.cantilever (reference test helper pattern)."""
    g = O.make_grid(dims)
    dpn = g.dpn
    ny = dims[1]
    if len(dims) == 2:
        left = [g.node_id(0, j) for j in range(ny + 1)]
    else:
        left = [g.node_id(0, j, k) for j in range(ny + 1) for k in range(dims[2] + 1)]
    fixed = np.unique(np.array([dpn * n + c for n in left for c in range(dpn)]))
    f = np.zeros(g.n_dofs)
    tip = g.node_id(*([dims[0]] + [d // 2 for d in dims[1:]]))
    f[dpn * tip + 1] = -1.0
    f[fixed] = 0.0
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.05, 1.0, g.n_elems)
    if void:
        rho = np.where(rng.uniform(size=g.n_elems) < 0.3, 1e-3, 1.0)
    E = O.simp_modulus(rho, 3.0, 1.0, 1e-9)
    K = O.assemble_stiffness(g, fixed, E)
    return g, fixed, f, rho, E, K


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_element_stiffness(golden):
    for tag, dims, h in (("q4", (1, 1), (1.0, 1.0)), ("q4h", (1, 1), (0.5, 0.25)),
                         ("hex8", (1, 1, 1), (1.0, 1.0, 1.0)),
                         ("hex8h", (1, 1, 1), (0.5, 0.5, 0.25))):
        ke = O.element_stiffness(O.make_grid(dims, h))
        assert np.max(np.abs(ke - golden["ke_" + tag])) <= 1e-14 * np.max(np.abs(ke))


def test_assembly_bc_rbm_filter(golden):
    g, fixed, f, rho, E, K = cantilever((6, 4), 1)
    assert np.array_equal(fixed, golden["asm_fixed"])
    assert np.array_equal(E, golden["asm_E"])
    assert np.max(np.abs(K.toarray() - golden["asm_K"])) <= 1e-15
    assert np.max(np.abs(O.rigid_body_modes(g, fixed) - golden["rbm_2d"])) <= 1e-15
    assert np.max(np.abs(O.rigid_body_modes(O.make_grid((3, 2, 2))) - golden["rbm_3d"])) <= 1e-15
    assert np.max(np.abs(O.density_filter(O.make_grid((5, 5))).toarray()
                         - golden["filter_5x5"])) <= 1e-15
    assert np.max(np.abs(O.density_filter(O.make_grid((3, 3, 2))).toarray()
                         - golden["filter_3d"])) <= 1e-15


@pytest.mark.parametrize("dims", [(4, 2), (5, 3), (6, 1), (4, 2, 2), (3, 2, 1)])
def test_geometric_prolongation_exact(golden, dims):
    P = O.geometric_prolongation(dims, len(dims)).toarray()
    assert np.array_equal(P, golden["P_" + "x".join(map(str, dims))])


def test_gmg_2d_hierarchy_vcycle_gmres(golden):
    g, fixed, f, rho, E, K = cantilever((16, 8), 2)
    assert np.array_equal(fixed, golden["gmg2d_fixed"])
    h = O.build_gmg(g, K, 60, O.Smoother("weighted_jacobi", 0.6), 2, 2)
    assert np.array_equal([lv.A.shape[0] for lv in h.levels], golden["gmg2d_sizes"])
    assert np.max(np.abs(h.levels[1].A.toarray() - golden["gmg2d_A1"])) <= 1e-13
    assert rel(h.apply(golden["gmg2d_b"]), golden["gmg2d_vc"]) <= 1e-12
    x, rec = O.gmres(K, f, None, h.apply, rtol=1e-8)
    assert np.array_equal(f, golden["gmg2d_f"])
    assert len(rec.residual_history) == len(golden["gmg2d_gmres_hist"])
    assert rel(x, golden["gmg2d_gmres_x"]) <= 1e-10
    x, rec = O.gmres(K, f, None, h.apply, rtol=1e-8, restart=5, flexible=True)
    assert len(rec.residual_history) == len(golden["gmg2d_fgmres_hist"])
    assert rel(x, golden["gmg2d_fgmres_x"]) <= 1e-10
    hb = O.build_gmg(g, K, 60, O.Smoother("block_jacobi", 0.5))
    assert rel(hb.apply(golden["gmg2d_b"]), golden["gmg2d_bj_vc"]) <= 1e-12


def test_gmg_3d_odd_dims(golden):
    g, fixed, f, rho, E, K = cantilever((5, 3, 3), 3)
    h = O.build_gmg(g, K, 50, O.Smoother("weighted_jacobi", 0.6), 1, 1)
    assert np.array_equal([lv.A.shape[0] for lv in h.levels], golden["gmg3d_sizes"])
    A = h.levels[-1].A.toarray()
    assert np.max(np.abs(A - golden["gmg3d_Alast"])) <= 1e-13 * np.max(np.abs(A))
    assert rel(h.apply(golden["gmg3d_b"]), golden["gmg3d_vc"]) <= 1e-12


@pytest.mark.parametrize("tag,dims,seed", [("sa2d", (12, 8), 4), ("sa3d", (6, 4, 4), 5)])
def test_sa_pieces_bit_exact(golden, tag, dims, seed):
    g, fixed, f, rho, E, K = cantilever(dims, seed, void=True)
    assert np.array_equal(E, golden[tag + "_E"])
    S = O.strength_graph(K, 0.08, g.dpn)
    assert np.array_equal(S.toarray(), golden[tag + "_S"])
    agg0, _ = O.aggregate(S)
    assert np.array_equal(agg0, golden[tag + "_agg0"])
    agg = O.merge_small(agg0, S, 2)
    assert np.array_equal(agg, golden[tag + "_agg"])
    T, Bc = O.tentative(agg, O.rigid_body_modes(g, fixed), g.dpn)
    assert np.max(np.abs(T.toarray() - golden[tag + "_T"])) <= 1e-13
    assert np.max(np.abs(Bc - golden[tag + "_Bc"])) <= 1e-12 * np.max(np.abs(Bc))
    P, omega = O.smooth_prolongation(K, T)
    assert np.max(np.abs(P.toarray() - golden[tag + "_P"])) <= 1e-12
    assert abs(O.spectral_radius(K) - float(golden[tag + "_rho"])) <= 1e-13
    h = O.build_sa_amg(K, O.rigid_body_modes(g, fixed), 40, O.Smoother(weight=0.6), 2, 2,
                       beta=0.003)
    h08 = O.build_sa_amg(K, O.rigid_body_modes(g, fixed), 40, O.Smoother(weight=0.6), 2, 2,
                         beta=0.003)
    assert h.n_levels == h08.n_levels


@pytest.mark.parametrize("tag,dims,seed", [("sa2d", (12, 8), 4), ("sa3d", (6, 4, 4), 5)])
def test_sa_hierarchy_vcycle(golden, tag, dims, seed):
    # make_golden builds these with the reference's fixed beta (0.003)
    g, fixed, f, rho, E, K = cantilever(dims, seed, void=True)
    h = O.build_sa_amg(K, O.rigid_body_modes(g, fixed), 40, O.Smoother(weight=0.6), 2, 2)
    assert np.array_equal([lv.A.shape[0] for lv in h.levels], golden[tag + "_sizes"])
    assert rel(h.apply(golden[tag + "_b"]), golden[tag + "_vc"]) <= 1e-10


def test_sa_default_and_forced(golden):
    g, fixed, f, rho, E, K = cantilever((12, 8), 4, void=True)
    h = O.build_sa_amg(K, O.rigid_body_modes(g, fixed), 40)
    assert np.array_equal([lv.A.shape[0] for lv in h.levels], golden["sa2d_default_sizes"])
    assert rel(h.apply(golden["sa2d_b"]), golden["sa2d_default_vc"]) <= 1e-10
    S = O.strength_graph(sp.identity(8, format="csr") * 3.0, block_size=1)
    agg, flags = O.aggregate(S)
    assert flags == ["forced_pairwise_aggregation"]
    assert np.array_equal(agg, golden["forced_agg"])


def test_hybrid_3d(golden):
    g, fixed, f, rho, E, K = cantilever((8, 4, 4), 6)
    h = O.build_hybrid(g, K, O.rigid_body_modes(g, fixed), 1, 60, O.Smoother(weight=0.6))
    assert np.array_equal([lv.A.shape[0] for lv in h.levels], golden["hyb3d_sizes"])
    assert np.array_equal([lv.provenance == "geometric" for lv in h.levels], golden["hyb3d_prov"])
    assert rel(h.apply(golden["hyb3d_b"]), golden["hyb3d_vc"]) <= 1e-10


def test_sensitivity(golden):
    g = O.make_grid((6, 4))
    ce = O.strain_energies(g, golden["sens_u"])
    assert rel(ce, golden["sens_ce"]) <= 1e-14
    dE = O.simp_derivative(golden["sens_rho"], 3.0, 1.0, 1e-9)
    assert rel(dE, golden["sens_dE"]) <= 1e-15
    g3 = O.make_grid((3, 2, 2))
    assert rel(O.strain_energies(g3, golden["sens3_u"]), golden["sens3_ce"]) <= 1e-14


def test_pcg_extension_matches_dense_solve():
    g, fixed, f, rho, E, K = cantilever((16, 8), 2)
    h = O.build_gmg(g, K, 60, O.Smoother("weighted_jacobi", 0.6), 2, 2)
    x, rec = O.pcg(K, f, None, h.apply, rtol=1e-10)
    xd = np.linalg.solve(K.toarray(), f)
    assert rec.converged and rel(x, xd) <= 1e-8
    assert np.linalg.norm(f - K @ x) <= 1e-10 * np.linalg.norm(f) * 1.01


def test_chebyshev_extension_reduces_error():
    g, fixed, f, rho, E, K = cantilever((8, 4), 3)
    sm = O.make_smoother(O.Smoother("chebyshev", inner_iterations=2), K)
    A = K.toarray()
    lam = np.linalg.eigvals(np.diag(1 / np.diag(A)) @ A).real.max()
    assert 0.5 * lam <= sm.lmax_estimate <= lam * (1 + 1e-12)
    xs = np.linalg.solve(A, f)
    x = sm.apply(np.zeros_like(f), f, 3)
    assert (xs - x) @ A @ (xs - x) < xs @ A @ xs


def test_sor_smoothers_gmg(golden):
    """SOR-Chebyshev / SOR-GMRES (multigrid.py:97-176) against the reference."""
    g, fixed, f, rho, E, K = cantilever((16, 8), 2)
    b = golden["sor2d_b"]
    for kind in ("sor_chebyshev", "sor_gmres"):
        h = O.build_gmg(g, K, 60, O.Smoother(kind), 1, 1)
        assert rel(h.apply(b), golden["sor2d_%s_vc" % kind]) <= 1e-11
        if kind == "sor_chebyshev":
            lm = [lv.smoother.lmax_estimate for lv in h.levels[:-1]]
            assert rel(lm, golden["sor2d_lmax"]) <= 1e-13
        sm = O.make_smoother(O.Smoother(kind, inner_iterations=3), K)
        assert rel(sm.apply(np.zeros_like(b), b, 2), golden["sor2d_%s_smooth" % kind]) <= 1e-11
    h = O.build_gmg(g, K, 60, O.Smoother("sor_gmres"))
    x, rec = O.gmres(K, f, None, h.apply, rtol=1e-8, flexible=True)
    assert len(rec.residual_history) == len(golden["sor2d_fgmres_hist"])
    assert rel(x, golden["sor2d_fgmres_x"]) <= 1e-9


def test_sor_and_block_jacobi_sa(golden):
    g, fixed, f, rho, E, K = cantilever((12, 8), 4, void=True)
    B = O.rigid_body_modes(g, fixed)
    for kind in ("sor_chebyshev", "sor_gmres", "block_jacobi"):
        h = O.build_sa_amg(K, B, 40, O.Smoother(kind, 0.6), 1, 1)
        assert rel(h.apply(golden["sorsa_b"]), golden["sorsa_%s_vc" % kind]) <= 1e-10


def test_sor_chebyshev_3d(golden):
    g, fixed, f, rho, E, K = cantilever((5, 3, 3), 3)
    h = O.build_gmg(g, K, 50, O.Smoother("sor_chebyshev"), 1, 1)
    lm = [lv.smoother.lmax_estimate for lv in h.levels[:-1]]
    assert rel(lm, golden["sor3d_lmax"]) <= 1e-13
    assert rel(h.apply(golden["sor3d_b"]), golden["sor3d_vc"]) <= 1e-11
