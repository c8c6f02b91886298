"""The host-buffer drop-in entry tmg_solve_compliance_host (the whole
compliance_and_sensitivity solve, optimization.py:114-133, numpy in / numpy out,
no PyTorch on the caller's side) for every Krylov method of krylov.solve and
every preconditioner strategy, against the CPU oracle."""

import ctypes as C

import numpy as np
import pytest

from oracle import topomg_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from bench import LegRunner  # noqa: E402
from paper_2001_01655_b200 import _lib, problems  # noqa: E402


def host_solve(w, leg, method, restart=0):
    L = _lib.load()
    law_p, e0, emin = problems.PENAL, problems.E0, problems.EMIN
    rho = np.ascontiguousarray(w.rho, dtype=np.float64)
    f = np.ascontiguousarray(w.bc.load_vector)
    fixed = np.ascontiguousarray(w.bc.fixed_dofs, dtype=np.int64)
    u = np.empty(w.ndof)
    dc = np.empty(w.mesh.element_count)
    comp = C.c_double()
    rec = _lib.SolveRec()
    md = _lib.mesh_desc(w.mesh)
    mg, keep = LegRunner(w, leg).mg_desc()
    cfg = _lib.SolveDesc(w.rtol, 500, method, restart)
    _lib.check(L.tmg_solve_compliance_host(C.byref(md), rho.ctypes.data, fixed.ctypes.data, fixed.size,
                                           f.ctypes.data, law_p, e0, emin, 0.3, C.byref(mg), C.byref(cfg),
                                           u.ctypes.data, dc.ctypes.data, C.byref(comp), C.byref(rec)))
    return u, dc, comp.value, rec


@pytest.mark.parametrize("method", [0, 1, 2])
def test_host_entry_gmg_all_methods(method):
    w = problems.config_0()
    leg = w.solvers[0]
    u, dc, comp, rec = host_solve(w, leg, method, restart=0 if method < 2 else 7)
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, problems.PENAL, problems.E0, problems.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    h = O.build_gmg(g, K, 1, O.Smoother("weighted_jacobi", 0.6), 2, 2, max_levels=3)
    f = w.bc.load_vector
    if method == 0:
        uo, ro = O.pcg(K, f, None, h.apply, rtol=w.rtol, max_iterations=500)
    else:
        uo, ro = O.gmres(K, f, None, h.apply, rtol=w.rtol, max_iterations=500,
                         restart=200 if method == 1 else 7, flexible=method == 2)
    assert rec.converged and ro.converged
    assert abs(rec.iterations - ro.iterations) <= 1
    assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
    Fo, dco = O.compliance_sensitivity(g, f, uo, w.rho, problems.PENAL, problems.E0, problems.EMIN)
    assert abs(comp - Fo) <= 1e-10 * abs(Fo)
    assert np.linalg.norm(dc - dco) <= 1e-8 * np.linalg.norm(dco)


def test_host_entry_rejects_unknown_method():
    w = problems.config_0()
    with pytest.raises(ValueError):
        host_solve(w, w.solvers[0], 5)


def _uniform_3d(dims=(16, 8, 8)):
    mesh, bc = problems._cantilever3d(*dims)
    rho = np.full(mesh.element_count, 0.5)
    return problems.Workload("cantilever3d_uniform", mesh, bc, rho)


@pytest.mark.parametrize("strategy", ["amg", "hybrid"])
def test_host_entry_amg_and_hybrid(strategy):
    """tmg_solve_compliance_host with the SA-AMG (2D MBB, config 0's mesh) and
    hybrid (3D cantilever, 1 geometric level then SA) strategies, PCG, against
    the oracle's compliance_and_sensitivity on the same hierarchy settings."""
    if strategy == "amg":
        w = problems.config_0()
        leg = dict(strategy="amg", coarse_max_dofs=499, beta=problems.BETA, isolated="drop",
                   smoother="weighted_jacobi", weight=0.6, n_pre=2, n_post=2)
    else:
        w = _uniform_3d()
        leg = dict(strategy="hybrid", n_geo=1, coarse_max_dofs=60, beta=problems.BETA, isolated="drop",
                   smoother="chebyshev", degree=2, lanczos_steps=10, n_pre=1, n_post=1)
    u, dc, comp, rec = host_solve(w, leg, 0)
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, problems.PENAL, problems.E0, problems.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    B = O.rigid_body_modes(g, w.bc.fixed_dofs)
    if strategy == "amg":
        h = O.build_sa_amg(K, B, 499, O.Smoother("weighted_jacobi", 0.6), 2, 2, beta=problems.BETA, isolated="drop")
    else:
        h = O.build_hybrid(g, K, B, 1, 60, O.Smoother("chebyshev", 1.0, 2, lanczos_steps=10), 1, 1,
                           beta=problems.BETA, isolated="drop")
    f = w.bc.load_vector
    uo, ro = O.pcg(K, f, None, h.apply, rtol=w.rtol, max_iterations=500)
    assert rec.converged and ro.converged
    assert abs(rec.iterations - ro.iterations) <= 1
    assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
    Fo, dco = O.compliance_sensitivity(g, f, uo, w.rho, problems.PENAL, problems.E0, problems.EMIN)
    assert abs(comp - Fo) <= 1e-10 * abs(Fo)
    assert np.linalg.norm(dc - dco) <= 1e-8 * np.linalg.norm(dco)


def test_host_entry_routes_sor_smoothers_to_fgmres():
    """optimization.py:90-95 through the C entry: method gmres with the
    non-stationary sor_gmres smoother runs FGMRES (matches the oracle's FGMRES),
    and the PCG extension refuses it (TMG_EINVAL -> ValueError)."""
    w = problems.config_0()
    leg = dict(strategy="gmg", levels=3, smoother="sor_gmres", weight=0.5, n_pre=1, n_post=1)
    u, dc, comp, rec = host_solve(w, leg, 1)
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, problems.PENAL, problems.E0, problems.EMIN)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    h = O.build_gmg(g, K, 1, O.Smoother("sor_gmres", 0.5), 1, 1, max_levels=3)
    uo, ro = O.gmres(K, w.bc.load_vector, None, h.apply, rtol=w.rtol, max_iterations=500, flexible=True)
    assert rec.converged and ro.converged
    assert abs(rec.iterations - ro.iterations) <= 1
    assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
    with pytest.raises(ValueError):
        host_solve(w, leg, 0)
