"""Solver harness and compliance sensitivity on the B200 (mirrors reference
optimization.py:36-132 for the compliance path)."""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, krylov
from ._dev import as_dev, empty_dev, ptr, stream_ptr
from .mesh import assemble_stiffness, rigid_body_modes
from .multigrid import (DEFAULT_STRENGTH_BETA, AdaptiveHybridController, SmootherConfig, adapt_after_solve,
                        build_gmg, build_hybrid, build_sa_amg, gmg_level_dims)


@dataclass
class SolverHarness:
    """Builds a multigrid preconditioner for each operator and runs the Krylov
    solve on the device (optimization.py:37).  strategy: 'gmg' | 'amg' |
    'hybrid' | 'hybrid_adaptive' | 'none'; the adaptive variant demotes one
    geometric level after a solve that needed more than 200 iterations
    (multigrid.py:614-631).  Extensions: n_pre/n_post/max_levels/beta/isolated
    (the reference uses the builders' defaults)."""

    mesh: object
    strategy: str = "amg"
    coarse_max_dofs: int = 200
    n_geo: int = 2
    smoother: SmootherConfig = field(default_factory=SmootherConfig)
    solve_cfg: krylov.SolveConfig = field(default_factory=krylov.SolveConfig)
    fixed_dofs: np.ndarray | None = None
    seed: int = 0
    n_pre: int = 1
    n_post: int = 1
    max_levels: int | None = None
    beta: float = DEFAULT_STRENGTH_BETA
    isolated: str = "merge"
    controller: AdaptiveHybridController | None = None

    def __post_init__(self):
        if self.strategy == "hybrid_adaptive" and self.controller is None:
            n_levels = len(gmg_level_dims(self.mesh.dims, self.mesh.dofs_per_node, self.coarse_max_dofs))
            start = max(2, min(self.n_geo, n_levels - 1))
            self.controller = AdaptiveHybridController(n_geo_current=start)

    @property
    def near_nullspace(self):
        return rigid_body_modes(self.mesh, self.fixed_dofs)

    def build(self, K):
        torch_sync()
        t0 = time.perf_counter()
        if self.strategy == "none":
            return None, 0.0
        if self.strategy == "gmg":
            h = build_gmg(self.mesh, K, self.coarse_max_dofs, self.smoother, self.n_pre, self.n_post,
                          self.max_levels)
        elif self.strategy == "amg":
            h = build_sa_amg(K, self.near_nullspace, self.coarse_max_dofs, self.smoother, self.n_pre,
                             self.n_post, seed=self.seed, beta=self.beta,
                             isolated=self.isolated)
        elif self.strategy in ("hybrid", "hybrid_adaptive"):
            n_geo = self.n_geo if self.strategy == "hybrid" else self.controller.n_geo_current
            h = build_hybrid(self.mesh, K, self.near_nullspace, n_geo, self.coarse_max_dofs,
                             self.smoother, self.n_pre, self.n_post, seed=self.seed, beta=self.beta,
                             isolated=self.isolated)
        else:
            raise ValueError("unknown preconditioner strategy %r" % self.strategy)
        torch_sync()
        return h, time.perf_counter() - t0

    def solve(self, K, f, x0=None, hierarchy=None):
        """Solve K x = f; returns (x, SolveRecord, hierarchy) (optimization.py:85).
        As the reference (optimization.py:90-95): GMRES for a stationary
        preconditioner unless FGMRES is asked for, FGMRES otherwise (the
        sor_chebyshev / sor_gmres smoothers).  method="cg" (the north-star PCG)
        needs a stationary symmetric V-cycle and is refused for the others."""
        setup = 0.0
        if hierarchy is None and self.strategy != "none":
            hierarchy, setup = self.build(K)
        stationary = hierarchy is None or hierarchy.stationary
        method = self.solve_cfg.method
        if method == "cg":
            if not stationary:
                raise ValueError("method='cg' needs a stationary preconditioner; the %s smoother is not "
                                 "(use 'gmres' -> FGMRES, as the reference)" % hierarchy.smoother_config.kind)
            x, rec = krylov.cg_solve(K, f, x0, hierarchy, self.solve_cfg)
        elif method not in ("gmres", "fgmres"):
            raise ValueError("unknown Krylov method %r" % method)
        elif stationary and method != "fgmres":
            x, rec = krylov.gmres_solve(K, f, x0, hierarchy, self.solve_cfg)
        else:
            x, rec = krylov.fgmres_solve(K, f, x0, hierarchy, self.solve_cfg)
        rec.setup_time = setup
        if self.strategy == "hybrid_adaptive":
            adapt_after_solve(self.controller, rec.iterations)
        return x, rec, hierarchy


def torch_sync():
    import torch
    torch.cuda.synchronize()


def element_strain_energies(mesh, u, ke=None, K=None):
    """u_e^T KE u_e with the unit-modulus KE (optimization.py:106), on the device."""
    if K is None:
        K = assemble_stiffness(mesh, None, np.ones(mesh.element_count))
    u = as_dev(u)
    out = empty_dev(mesh.element_count)
    _lib.check(_lib.load().tmg_strain_energy(K.handle, ptr(u), ptr(out), stream_ptr(None)))
    return out


def compliance_and_sensitivity(mesh, bc, filt, law, alpha, harness, u0=None):
    """F = f^T u and dF/dalpha (optimization.py:114).  filt: object with
    apply/apply_transpose (host) or None when alpha is already rho."""
    rho = filt.apply(alpha) if filt is not None else np.asarray(alpha, dtype=float)
    E = law.modulus(rho)
    K = assemble_stiffness(mesh, bc, E)
    u, rec, hierarchy = harness.solve(K, bc.load_vector, u0)
    if not rec.converged:
        raise RuntimeError("displacement solve failed to converge (%d iterations, final residual %.3e)"
                           % (rec.iterations, rec.residual_history[-1]))
    rho_d = as_dev(rho)
    f_d = as_dev(bc.load_vector)
    dc = empty_dev(mesh.element_count)
    comp = C.c_double()
    _lib.check(_lib.load().tmg_compliance_sensitivity(
        K.handle, ptr(rho_d), ptr(f_d), ptr(u), float(law.penalty), float(law.e_max), float(law.e_min),
        ptr(dc), C.byref(comp), stream_ptr(None)))
    dF_drho = dc.cpu().numpy()
    dF = filt.apply_transpose(dF_drho) if filt is not None else dF_drho
    aux = {"u": u, "K": K, "record": rec, "hierarchy": hierarchy, "rho": rho}
    return comp.value, dF, aux
