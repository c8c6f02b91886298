"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
host-only entry points agree with the reference golden vectors, and the host
input generators agree with the oracle.  No GPU needed."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import topomg_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def lib():
    from paper_2001_01655_b200 import _lib
    return _lib


def test_library_exports_every_header_symbol():
    L = lib()
    handle = L.load()
    header = open(os.path.join(ROOT, "include", "topomg_b200.h")).read()
    declared = set(re.findall(r"\b(tmg_[a-z_0-9]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(handle, name), name
    assert declared == set(L.EXPORTS)
    assert handle.tmg_version() >= 100


def test_no_device_reports_enodev_not_fallback():
    L = lib()
    if L.load().tmg_device_count() > 0:
        pytest.skip("GPU present")
    out = C.c_void_p()
    mesh = L.MeshDesc(2, (C.c_int32 * 3)(2, 1, 1), (C.c_double * 3)(1, 1, 1))
    rc = L.load().tmg_operator_create(C.byref(mesh), None, None, 0, 0.3, None, C.byref(out))
    assert rc == L.TMG_ENODEV


@pytest.mark.parametrize("tag,dims,h", [("q4", (1, 1), (1.0, 1.0)), ("q4h", (1, 1), (0.5, 0.25)),
                                        ("hex8", (1, 1, 1), (1.0, 1.0, 1.0)),
                                        ("hex8h", (1, 1, 1), (0.5, 0.5, 0.25))])
def test_native_element_stiffness_matches_reference(golden, tag, dims, h):
    from paper_2001_01655_b200.mesh import build_mesh, element_stiffness
    ke = element_stiffness(build_mesh(dims, h))
    ref = golden["ke_" + tag]
    assert np.max(np.abs(ke - ref)) <= 1e-14 * np.max(np.abs(ref))


def test_element_stiffness_validation():
    from paper_2001_01655_b200.mesh import build_mesh, element_stiffness
    with pytest.raises(ValueError):
        element_stiffness(build_mesh((1, 1)), 1.0, 0.5)
    with pytest.raises(ValueError):
        element_stiffness(build_mesh((1, 1)), -1.0, 0.3)
    with pytest.raises(ValueError):
        build_mesh((2, 0))


def test_mesh_numbering_matches_oracle():
    from paper_2001_01655_b200.mesh import build_mesh
    for dims in ((3, 2), (2, 3, 2)):
        m, g = build_mesh(dims), O.make_grid(dims)
        assert np.array_equal(m.element_dofs(), g.edofs())
        assert np.array_equal(m.node_coordinates(), g.coords())


def test_cone_filter_equals_reference_filter_matrix():
    from paper_2001_01655_b200.problems import cone_filter, to_elements
    rng = np.random.default_rng(0)
    for shape in ((7, 5), (4, 3, 5)):
        a = rng.uniform(size=shape)
        S = O.density_filter(O.make_grid(shape), 1.5)
        assert np.max(np.abs(to_elements(cone_filter(a)) - S @ to_elements(a))) <= 1e-14


def test_gmg_plan_matches_oracle():
    from paper_2001_01655_b200.multigrid import gmg_level_dims
    for dims, bound in (((2048, 1024), 150), ((960, 320), 5000), ((5, 3, 3), 50)):
        assert gmg_level_dims(dims, len(dims), bound) == O.gmg_plan(dims, len(dims), bound)
    assert len(gmg_level_dims((960, 320), 2, 1, max_levels=5)) == 5


def test_workload_generators():
    from paper_2001_01655_b200 import problems
    w = problems.config_0()
    assert w.ndof == 9922 and np.all(w.rho == 0.5)
    assert w.bc.load_vector.sum() == -1.0
    w1 = problems.config_1()
    assert w1.ndof == 961 * 321 * 2  # BASELINE.json quotes 617,442; (nx+1)(ny+1)*2 is exact
    assert set(np.unique(w1.rho)) >= {1.0, problems.VOID}
    assert 0.3 < w1.rho.mean() < 0.5
    w3 = problems.config_3()
    assert w3.ndof == 97 * 49 * 49 * 3 and abs(w3.bc.load_vector.sum() + 1.0) < 1e-12


def test_adaptive_hybrid_controller_host_logic():
    """multigrid.py:614-631: demote one geometric level after a >200-iteration
    solve, never below min_geo."""
    from paper_2001_01655_b200 import AdaptiveHybridController, adapt_after_solve
    c = AdaptiveHybridController(n_geo_current=3)
    assert adapt_after_solve(c, 150) == "keep" and c.n_geo_current == 3
    assert adapt_after_solve(c, 201) == "rebuild" and c.n_geo_current == 2
    assert adapt_after_solve(c, 500) == "keep" and c.n_geo_current == 2
    with pytest.raises(ValueError):
        AdaptiveHybridController(n_geo_current=1)


def test_solve_config_validation_and_methods():
    from paper_2001_01655_b200 import SolveConfig
    # the reference's defaults (krylov.py:17-19); the north-star PCG is opt-in
    assert (SolveConfig().method, SolveConfig().rtol, SolveConfig().restart) == ("gmres", 1e-7, 200)
    for bad in (dict(rtol=0.0), dict(rtol=1.0), dict(restart=0)):
        with pytest.raises(ValueError):
            SolveConfig(**bad)


def test_smoother_descriptor_host_logic():
    """SmootherConfig -> tmg_smoother_desc: every reference kind is known, the
    sor_chebyshev descriptor carries multigrid.py:119's power-method start vector
    (default_rng(0), the smoother is built with seed 0) for the finest level."""
    from paper_2001_01655_b200 import SmootherConfig
    from paper_2001_01655_b200.multigrid import SMOOTHER_KINDS
    assert set(SMOOTHER_KINDS) >= {"weighted_jacobi", "block_jacobi", "sor_chebyshev", "sor_gmres"}
    d = SmootherConfig(kind="sor_chebyshev", inner_iterations=3).desc(257)
    assert d.kind == SMOOTHER_KINDS["sor_chebyshev"] and d.inner_iterations == 3
    ps = np.ctypeslib.as_array((C.c_double * 257).from_address(d.power_start))
    assert np.array_equal(ps, np.random.default_rng(0).standard_normal(257))
    assert not SmootherConfig(kind="sor_gmres").desc(10).power_start
    assert not SmootherConfig(kind="sor_gmres").stationary and SmootherConfig().stationary
    assert not SmootherConfig(kind="sor_chebyshev").stationary
    assert SmootherConfig(kind="chebyshev", weight=1.0).stationary  # fixed polynomial in D^-1 A
    with pytest.raises(ValueError):
        SmootherConfig(kind="sor").desc(10)
    with pytest.raises(ValueError):
        SmootherConfig(weight=0.0)


def test_solve_descriptor_defaults_to_cg():
    """tmg_solve_desc zero-initialised fields keep the CG extension; method/restart
    select krylov.solve's GMRES / FGMRES in the host-buffer entry."""
    L = lib()
    d = L.SolveDesc(1e-8, 100)
    assert (d.method, d.restart) == (0, 0)
    d = L.SolveDesc(1e-8, 100, 2, 7)
    assert (d.method, d.restart) == (2, 7)


def test_harness_routes_like_the_reference(monkeypatch):
    """optimization.py:90-95: GMRES for a stationary preconditioner unless FGMRES
    is asked for, FGMRES for the SOR smoothers; method="cg" refuses a
    non-stationary V-cycle (host logic only, the Krylov drivers are stubbed)."""
    import paper_2001_01655_b200 as T
    from paper_2001_01655_b200 import krylov

    calls = []
    for name in ("cg_solve", "gmres_solve", "fgmres_solve"):
        monkeypatch.setattr(krylov, name, lambda *a, _n=name, **k: (calls.append(_n) or (None, krylov.SolveRecord())))

    class H:
        def __init__(self, kind):
            self.smoother_config = T.SmootherConfig(kind=kind)

        @property
        def stationary(self):
            return self.smoother_config.stationary

    mesh = T.build_mesh((4, 2))
    for kind, method, want in (("weighted_jacobi", "gmres", "gmres_solve"), ("weighted_jacobi", "fgmres", "fgmres_solve"),
                               ("sor_gmres", "gmres", "fgmres_solve"), ("sor_chebyshev", "gmres", "fgmres_solve"),
                               ("weighted_jacobi", "cg", "cg_solve")):
        hs = T.SolverHarness(mesh, strategy="gmg", solve_cfg=T.SolveConfig(method=method))
        calls.clear()
        hs.solve(None, None, hierarchy=H(kind))
        assert calls == [want], (kind, method, calls)
    hs = T.SolverHarness(mesh, strategy="gmg", solve_cfg=T.SolveConfig(method="cg"))
    with pytest.raises(ValueError):
        hs.solve(None, None, hierarchy=H("sor_gmres"))
    hs = T.SolverHarness(mesh, strategy="none", solve_cfg=T.SolveConfig())
    calls.clear()
    hs.solve(None, None)
    assert calls == ["gmres_solve"]
