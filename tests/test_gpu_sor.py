"""SOR smoothers (multigrid.py:97-176: sor_chebyshev, sor_gmres) and block
Jacobi on smoothed-aggregation levels (multigrid.py:64 with block_size = nvec)
on the device, against the reference's golden vectors and the oracle."""

import numpy as np
import pytest

from oracle import topomg_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2001_01655_b200 as T  # noqa: E402
from test_gpu_parity import cantilever, host, rel  # noqa: E402
from test_oracle_golden import cantilever as golden_cantilever  # noqa: E402


def _device_problem(dims, seed, void=False):
    g, fixed, f, rho, E, Kref = golden_cantilever(dims, seed, void)
    mesh = T.build_mesh(dims)
    bc = T.BoundaryConditions(fixed, f)
    return mesh, bc, g, fixed, f, E, T.assemble_stiffness(mesh, bc, E), Kref


@pytest.mark.parametrize("kind", ["sor_chebyshev", "sor_gmres"])
def test_sor_gmg_vcycle_matches_reference_golden(golden, kind):
    mesh, bc, g, fixed, f, E, K, Kref = _device_problem((16, 8), 2)
    h = T.build_gmg(mesh, K, 60, T.SmootherConfig(kind=kind), 1, 1)
    assert rel(host(h.apply(golden["sor2d_b"])), golden["sor2d_%s_vc" % kind]) <= 1e-9
    if kind == "sor_chebyshev":
        lm = [h.level_lmax(k) for k in range(h.n_levels - 1)]
        assert rel(lm, golden["sor2d_lmax"]) <= 1e-10


def test_fgmres_with_sor_gmres_vcycle_matches_reference_golden(golden):
    """reference test_krylov.py:67 setting: FGMRES preconditioned by a GMG V-cycle
    with the SOR-GMRES smoother."""
    mesh, bc, g, fixed, f, E, K, Kref = _device_problem((16, 8), 2)
    h = T.build_gmg(mesh, K, 60, T.SmootherConfig(kind="sor_gmres"))
    x, rec = T.solve(K, f, None, h, T.SolveConfig(method="fgmres", rtol=1e-8))
    ref_hist = golden["sor2d_fgmres_hist"]
    assert rec.converged
    assert abs(len(rec.residual_history) - len(ref_hist)) <= 1
    assert rel(host(x), golden["sor2d_fgmres_x"]) <= 1e-8


@pytest.mark.parametrize("kind", ["sor_chebyshev", "sor_gmres", "block_jacobi"])
def test_sa_smoothers_match_reference_golden(golden, kind):
    mesh, bc, g, fixed, f, E, K, Kref = _device_problem((12, 8), 4, void=True)
    B = T.rigid_body_modes(mesh, fixed)
    h = T.build_sa_amg(K, B, 40, T.SmootherConfig(kind=kind, weight=0.6), 1, 1)
    assert rel(host(h.apply(golden["sorsa_b"])), golden["sorsa_%s_vc" % kind]) <= 1e-9


def test_sor_chebyshev_3d_matches_reference_golden(golden):
    mesh, bc, g, fixed, f, E, K, Kref = _device_problem((5, 3, 3), 3)
    h = T.build_gmg(mesh, K, 50, T.SmootherConfig(kind="sor_chebyshev"), 1, 1)
    lm = [h.level_lmax(k) for k in range(h.n_levels - 1)]
    assert rel(lm, golden["sor3d_lmax"]) <= 1e-10
    assert rel(host(h.apply(golden["sor3d_b"])), golden["sor3d_vc"]) <= 1e-9


@pytest.mark.parametrize("dims,kind,inner,passes", [((32, 16), "sor_gmres", 3, 2), ((32, 16), "sor_chebyshev", 3, 2),
                                                    ((8, 4, 4), "sor_gmres", 2, 1)])
def test_sor_gmg_matches_oracle(dims, kind, inner, passes):
    mesh, g, bc, rho, E, K, Kref = cantilever(dims, 5)
    h = T.build_gmg(mesh, K, 60, T.SmootherConfig(kind=kind, inner_iterations=inner), passes, passes)
    ho = O.build_gmg(g, Kref, 60, O.Smoother(kind, inner_iterations=inner), passes, passes)
    b = np.random.default_rng(9).standard_normal(g.n_dofs)
    assert rel(host(h.apply(b)), ho.apply(b)) <= 1e-9
    x, rec = T.solve(K, bc.load_vector, None, h, T.SolveConfig(method="fgmres", rtol=1e-8, max_iterations=300))
    xo, reco = O.gmres(Kref, bc.load_vector, None, ho.apply, rtol=1e-8, flexible=True, max_iterations=300)
    assert rec.converged and reco.converged
    assert abs(rec.iterations - reco.iterations) <= 1
    assert rel(host(x), xo) <= 1e-8


@pytest.mark.parametrize("kind", ["sor_chebyshev", "sor_gmres", "block_jacobi"])
def test_sor_hybrid_3d_matches_oracle(kind):
    mesh, g, bc, rho, E, K, Kref = cantilever((8, 4, 4), 6)
    B = T.rigid_body_modes(mesh, bc.fixed_dofs)
    sm = T.SmootherConfig(kind=kind, weight=0.6)
    h = T.build_hybrid(mesh, K, B, 1, 60, sm, 1, 1)
    ho = O.build_hybrid(g, Kref, O.rigid_body_modes(g, bc.fixed_dofs), 1, 60, O.Smoother(kind, 0.6), 1, 1)
    assert [lv.size for lv in h.levels] == [lv.A.shape[0] for lv in ho.levels]
    b = np.random.default_rng(2).standard_normal(g.n_dofs)
    assert rel(host(h.apply(b)), ho.apply(b)) <= 1e-9


def test_sor_vcycle_is_deterministic():
    """The sync-free triangular solve fixes each row's summation order, so two
    applications agree bit for bit."""
    mesh, g, bc, rho, E, K, Kref = cantilever((24, 12), 7)
    h = T.build_gmg(mesh, K, 60, T.SmootherConfig(kind="sor_gmres"), 2, 2)
    b = torch.as_tensor(np.random.default_rng(3).standard_normal(g.n_dofs), device="cuda")
    a1, a2 = host(h.apply(b)), host(h.apply(b))
    assert np.array_equal(a1, a2)


@pytest.mark.parametrize("kind", ["sor_chebyshev", "sor_gmres"])
def test_standalone_sor_smooth_matches_reference_golden(golden, kind):
    """multigrid.smooth(SmootherConfig(kind, inner_iterations=3), K, 0, b, passes=2)
    as the reference ran it in make_golden.py."""
    mesh, bc, g, fixed, f, E, K, Kref = _device_problem((16, 8), 2)
    x = T.smooth(T.SmootherConfig(kind=kind, inner_iterations=3), K, np.zeros(K.shape[0]), golden["sor2d_b"], passes=2)
    assert rel(host(x), golden["sor2d_%s_smooth" % kind]) <= 1e-9


@pytest.mark.parametrize("dims,kind", [((24, 12), "weighted_jacobi"), ((24, 12), "block_jacobi"),
                                       ((24, 12), "chebyshev"), ((24, 12), "sor_chebyshev"),
                                       ((24, 12), "sor_gmres"), ((6, 4, 4), "weighted_jacobi"),
                                       ((6, 4, 4), "block_jacobi"), ((6, 4, 4), "sor_chebyshev"),
                                       ((6, 4, 4), "sor_gmres")])
def test_standalone_smoothers_match_oracle(dims, kind):
    """make_smoother(config, K).apply(x, b, passes) (multigrid.py:179) from a
    nonzero start, against the oracle's smoother classes."""
    mesh, g, bc, rho, E, K, Kref = cantilever(dims, 4)
    w = 1.0 if kind == "chebyshev" else 0.6
    sm = T.make_smoother(T.SmootherConfig(kind=kind, weight=w, inner_iterations=2, block_size=len(dims)), K)
    so = O.make_smoother(O.Smoother(kind, w, inner_iterations=2, block_size=len(dims)), Kref)
    rng = np.random.default_rng(8)
    x0 = rng.standard_normal(g.n_dofs)
    x0[bc.fixed_dofs] = 0.0
    b = rng.standard_normal(g.n_dofs)
    x = host(sm.apply(x0, b, 3))
    xo = so.apply(x0.copy(), b, 3)
    assert rel(x, xo) <= 1e-9, kind
    if kind in ("chebyshev", "sor_chebyshev"):
        assert abs(sm.lmax_estimate - so.lmax_estimate) <= 1e-10 * so.lmax_estimate
    with pytest.raises(ValueError):  # a smoother is not a preconditioner
        sm.vcycle(b)
