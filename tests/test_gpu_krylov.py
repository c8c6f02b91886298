"""Device GMRES / flexible GMRES (krylov.py:48-146, the reference's default
Krylov method) against the reference's own golden vectors and the oracle."""

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


def test_gmres_matches_reference_golden(golden):
    """Same problem as the reference run in make_golden.py: (16, 8) cantilever,
    GMG 2/2 weighted Jacobi 0.6, rtol 1e-8; GMRES(200) and FGMRES(5)."""
    g, fixed, f, rho, E, Kref = golden_cantilever((16, 8), 2)
    mesh = T.build_mesh((16, 8))
    K = T.assemble_stiffness(mesh, T.BoundaryConditions(fixed, f), E)
    h = T.build_gmg(mesh, K, 60, T.SmootherConfig(weight=0.6), 2, 2)
    x, rec = T.solve(K, f, None, h, T.SolveConfig(method="gmres", rtol=1e-8))
    ref_hist = golden["gmg2d_gmres_hist"]
    assert rec.converged
    assert abs(len(rec.residual_history) - len(ref_hist)) <= 1          # iterations +-1
    assert rel(host(x), golden["gmg2d_gmres_x"]) <= 1e-8
    n = min(len(ref_hist), len(rec.residual_history)) - 1
    assert rel(rec.residual_history[:n], ref_hist[:n]) <= 1e-6            # history, before the rounding tail
    x, rec = T.solve(K, f, None, h, T.SolveConfig(method="fgmres", rtol=1e-8, restart=5))
    ref_hist = golden["gmg2d_fgmres_hist"]
    assert rec.converged
    assert abs(len(rec.residual_history) - len(ref_hist)) <= 1
    assert rel(host(x), golden["gmg2d_fgmres_x"]) <= 1e-8


@pytest.mark.parametrize("dims,restart,flexible", [((24, 12), 200, False), ((24, 12), 7, False),
                                                   ((8, 4, 4), 10, True), ((6, 4, 4), 200, False)])
def test_gmres_matches_oracle(dims, restart, flexible):
    mesh, g, bc, rho, E, K, Kref = cantilever(dims, 3)
    sm = T.SmootherConfig(weight=0.6)
    h = T.build_gmg(mesh, K, 60, sm, 1, 1)
    ho = O.build_gmg(g, Kref, 60, O.Smoother(weight=0.6), 1, 1)
    method = "fgmres" if flexible else "gmres"
    x, rec = T.solve(K, bc.load_vector, None, h, T.SolveConfig(method=method, rtol=1e-8, restart=restart,
                                                               max_iterations=500))
    xo, reco = O.gmres(Kref, bc.load_vector, None, ho.apply, rtol=1e-8, restart=restart, flexible=flexible,
                       max_iterations=500)
    assert rec.converged and reco.converged
    assert abs(rec.iterations - reco.iterations) <= 1
    assert rel(host(x), xo) <= 1e-8
    f = bc.load_vector
    assert abs(f @ host(x) - f @ xo) <= 1e-10 * abs(f @ xo)


def test_gmres_unpreconditioned_warm_start_and_cap():
    mesh, g, bc, rho, E, K, Kref = cantilever((10, 5), 4)
    f = bc.load_vector
    x, rec = T.solve(K, f, None, None, T.SolveConfig(method="gmres", rtol=1e-9, max_iterations=400))
    xo, reco = O.gmres(Kref, f, None, None, rtol=1e-9, max_iterations=400)
    assert abs(rec.iterations - reco.iterations) <= 1 and rec.converged == reco.converged
    # warm start at the solution: zero iterations, converged (krylov.py:64-68)
    x2, rec2 = T.solve(K, f, host(x), None, T.SolveConfig(method="gmres", rtol=1e-6))
    assert rec2.iterations == 0 and rec2.converged
    # iteration cap: stops at max_iterations, not converged
    x3, rec3 = T.solve(K, f, None, None, T.SolveConfig(method="gmres", rtol=1e-12, max_iterations=7, restart=3))
    assert rec3.iterations == 7 and not rec3.converged
    assert len(rec3.residual_history) == 8


def test_harness_dispatches_methods_and_adapts():
    mesh, g, bc, rho, E, K, Kref = cantilever((16, 8), 5)
    hs = T.SolverHarness(mesh, strategy="gmg", coarse_max_dofs=60, fixed_dofs=bc.fixed_dofs,
                         solve_cfg=T.SolveConfig(method="gmres", rtol=1e-8))
    x, rec, h = hs.solve(K, bc.load_vector)
    assert rec.converged
    ha = T.SolverHarness(mesh, strategy="hybrid_adaptive", coarse_max_dofs=60, n_geo=3, fixed_dofs=bc.fixed_dofs,
                         solve_cfg=T.SolveConfig(method="cg", rtol=1e-8))
    start = ha.controller.n_geo_current
    x, rec, h = ha.solve(K, bc.load_vector)
    assert rec.converged
    assert ha.controller.n_geo_current == (start - 1 if rec.iterations > 200 and start > 2 else start)
    with pytest.raises(ValueError):
        T.solve(K, bc.load_vector, None, None, T.SolveConfig(method="bicgstab"))
