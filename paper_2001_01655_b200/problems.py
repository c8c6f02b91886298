"""Seeded synthetic workloads of BASELINE.json ``configs`` (host-side input
generation only; these are the inputs both the device path and the CPU oracle
consume).

Each ``config_N()`` returns a ``Workload`` with the mesh, boundary conditions,
load cases, density field and the solver/preconditioner settings the config
names.  Densities follow the config text: Gaussian random fields (FFT-free,
separable Gaussian smoothing of seeded white noise) thresholded at the stated
volume fraction to {1, 1e-3} and smoothed by the reference's linear cone filter
(mesh.py:369, row-normalised hat weights) -- seeded stand-ins for evolved
topologies, as DESIGN.md records.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import BoundaryConditions, build_mesh

E0, EMIN, NU, PENAL = 1.0, 1e-9, 0.3, 3.0
VOID = 1e-3
# "symmetric strength threshold 0.08" is theta in ||A_IJ|| > theta sqrt(||A_II|| ||A_JJ||);
# the reference's rule (multigrid.py:355) is the squared form ||A_IJ||^2 > beta ..., so
# beta = theta^2.  (beta = 0.08 literally would isolate 98% of config 1's nodes.)
THETA = 0.08
BETA = THETA * THETA
# Strength-isolated nodes (void nodes whose every coupling is below the threshold;
# 7059 of them on config 1) become singletons that the reference's fallback folds
# into ONE aggregate spanning the domain (multigrid.py:457-467); its Galerkin
# product fills in quadratically and the setup never finishes at BASELINE sizes.
# The bench legs therefore run isolated="drop" (PyAMG's treatment: unaggregated,
# zero rows of T); "merge" stays the default of the API and is parity-tested.


@dataclass
class Workload:
    name: str
    mesh: object
    bc: BoundaryConditions
    rho: np.ndarray
    loads: list = field(default_factory=list)      # extra load vectors (same BCs)
    solvers: list = field(default_factory=list)    # dicts: strategy + settings
    rtol: float = 1e-8

    @property
    def moduli(self):
        return EMIN + (E0 - EMIN) * self.rho ** PENAL

    @property
    def ndof(self):
        return self.mesh.total_dofs


def cone_filter(field_, radius=1.5):
    """Row-normalised hat filter w = max(0, r - d) over element centroids, the
    reference's build_filter (mesh.py:369) applied as a stencil."""
    ndim = field_.ndim
    reach = max(int(np.ceil(radius - 1e-12)) - 1, 0)
    num = np.zeros_like(field_, dtype=float)
    den = np.zeros_like(field_, dtype=float)
    ones = np.ones_like(field_, dtype=float)
    rng = range(-reach, reach + 1)
    offs = [(a, b) for a in rng for b in rng] if ndim == 2 else \
        [(a, b, c) for a in rng for b in rng for c in rng]
    for off in offs:
        d = float(np.sqrt(sum(o * o for o in off)))
        if d >= radius:
            continue
        w = radius - d
        src = [slice(max(0, o), n + min(0, o)) for o, n in zip(off, field_.shape)]
        dst = [slice(max(0, -o), n + min(0, -o)) for o, n in zip(off, field_.shape)]
        num[tuple(dst)] += w * field_[tuple(src)]
        den[tuple(dst)] += w * ones[tuple(src)]
    return num / den


def gaussian_field(shape, corr_len, seed):
    """Seeded Gaussian random field with Gaussian covariance of length corr_len."""
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal(shape)
    return gaussian_filter(noise, sigma=corr_len / np.sqrt(2.0), mode="reflect")


def threshold(field_, volfrac):
    cut = np.quantile(field_, 1.0 - volfrac)
    return np.where(field_ >= cut, 1.0, VOID)


def to_elements(arr):
    """(nx, ny[, nz]) array -> element vector with x fastest (mesh.py:73)."""
    return np.ascontiguousarray(arr).reshape(-1, order="F")


def _mbb(nx, ny):
    mesh = build_mesh((nx, ny))
    fixed = [2 * mesh.node_index(0, j) for j in range(ny + 1)]           # x-dofs, left edge
    fixed.append(2 * mesh.node_index(nx, 0) + 1)                         # y-dof, bottom-right
    f = np.zeros(mesh.total_dofs)
    f[2 * mesh.node_index(0, ny) + 1] = -1.0                             # top-left, downward
    return mesh, BoundaryConditions(np.array(fixed), f)


def config_0():
    mesh, bc = _mbb(120, 40)
    rho = np.full(mesh.element_count, 0.5)
    return Workload("mbb2d_120x40_gmg3", mesh, bc, rho,
                    solvers=[dict(strategy="gmg", levels=3, smoother="weighted_jacobi", weight=0.6,
                                  n_pre=2, n_post=2)])


def config_1(seed=1655, dims=(960, 320)):
    nx, ny = dims
    mesh, bc = _mbb(nx, ny)
    g = gaussian_field((nx, ny), 8.0, seed)
    rho = cone_filter(threshold(g, 0.4), 1.5)
    return Workload("mbb2d_960x320_gmg5_vs_amg", mesh, bc, to_elements(rho),
                    # omega=0.6 point Jacobi exceeds 2/lambda_max(D^-1 A) on the Galerkin
                    # levels 2-3 of this hierarchy (lambda 3.38, 3.51): the V-cycle is then
                    # indefinite and PCG cannot converge.  The bench leg caps the weight at
                    # 1.8/lambda_hat per level.
                    # The thresholded field does not percolate (128 solid islands in void,
                    # E contrast 5e8): GMG-PCG stagnates (rel. residual ~1e-4 after 20000
                    # iterations), so the bench caps this leg at 2000 iterations and
                    # reports the converged flag -- the paper's GMG failure mode.
                    solvers=[dict(strategy="gmg", levels=5, smoother="weighted_jacobi", weight=0.6,
                                  n_pre=2, n_post=2, safeguard=1.8, max_iterations=2000),
                             # (the same cap on the SA leg: w * lambda_max(D^-1 A) = 2.19 on its level 3)
                             dict(strategy="amg", coarse_max_dofs=499, beta=BETA, isolated="drop",
                                  smoother="weighted_jacobi", weight=0.6, n_pre=2, n_post=2, safeguard=1.8,
                                  max_iterations=2000)])


def config_2(seed=2001, dims=(1920, 640)):
    nx, ny = dims
    mesh = build_mesh((nx, ny))
    fixed = [2 * mesh.node_index(0, j) + c for j in range(ny + 1) for c in (0, 1)]
    rng = np.random.default_rng(seed)
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    solid = np.zeros((nx, ny), dtype=bool)
    for coord in (ix - iy, ix + iy):
        sid = np.floor_divide(coord, 24)
        ids = np.arange(sid.min(), sid.max() + 1)
        keep = rng.uniform(size=ids.size) < 0.85
        on = (np.mod(coord, 24) < 2) & keep[sid - ids[0]]
        solid |= on
    rho = np.where(solid, 1.0, VOID)
    loads = []
    for node, comp, val in ((mesh.node_index(nx, ny // 2), 1, -1.0), (mesh.node_index(nx, ny), 1, 1.0),
                            (mesh.node_index(nx, 0), 0, 1.0)):
        f = np.zeros(mesh.total_dofs)
        f[2 * node + comp] = val
        loads.append(f)
    f = np.zeros(mesh.total_dofs)
    right = np.array([mesh.node_index(nx, j) for j in range(ny + 1)])
    f[2 * right] = rng.uniform(-1, 1, right.size)
    f[2 * right + 1] = rng.uniform(-1, 1, right.size)
    loads.append(f)
    bc = BoundaryConditions(np.array(fixed), loads[0])
    return Workload("cantilever2d_1920x640_amg_4loads", mesh, bc, to_elements(rho), loads=loads[1:],
                    solvers=[dict(strategy="amg", coarse_max_dofs=499, beta=BETA, isolated="drop",
                                  smoother="weighted_jacobi", weight=0.6, n_pre=2, n_post=2)])


def _cantilever3d(nx, ny, nz):
    mesh = build_mesh((nx, ny, nz))
    fixed = [3 * mesh.node_index(0, j, k) + c for j in range(ny + 1) for k in range(nz + 1) for c in range(3)]
    f = np.zeros(mesh.total_dofs)
    w = np.ones(ny + 1)
    w[0] = w[-1] = 0.5
    w /= w.sum()
    for j in range(ny + 1):
        f[3 * mesh.node_index(nx, j, 0) + 2] = -w[j]
    return mesh, BoundaryConditions(np.array(fixed), f)


def config_3(seed=3003, dims=(96, 48, 48)):
    nx, ny, nz = dims
    mesh, bc = _cantilever3d(nx, ny, nz)
    g = gaussian_field((nx, ny, nz), 6.0, seed)
    rho = cone_filter(threshold(g, 0.15), 1.5)
    return Workload("cantilever3d_96x48x48_gmg4_cheb", mesh, bc, to_elements(rho),
                    solvers=[dict(strategy="gmg", levels=4, smoother="chebyshev", degree=2,
                                  lanczos_steps=10, n_pre=1, n_post=1)])


def config_4(seed=4004, dims=(192, 96, 96)):
    nx, ny, nz = dims
    mesh, bc = _cantilever3d(nx, ny, nz)
    g = gaussian_field((nx, ny, nz), 10.0, seed)
    rho = cone_filter(threshold(g, 0.12), 1.5)
    return Workload("cantilever3d_192x96x96_hybrid", mesh, bc, to_elements(rho),
                    solvers=[dict(strategy="hybrid", n_geo=3, coarse_max_dofs=999, beta=BETA, isolated="drop",
                                  smoother="chebyshev", degree=2, lanczos_steps=10, n_pre=1, n_post=1)])


CONFIGS = {0: config_0, 1: config_1, 2: config_2, 3: config_3, 4: config_4}


def leg_name(solver):
    s = solver["strategy"]
    if s == "gmg":
        return "gmg%d" % solver["levels"]
    if s == "hybrid":
        return "hybrid%d+amg" % solver["n_geo"]
    return "amg"


def smoother_settings(solver):
    return gmg_settings(solver)


def gmg_settings(solver):
    """SmootherConfig for a solver entry of a workload."""
    from .multigrid import SmootherConfig
    if solver["smoother"] == "chebyshev":
        sm = SmootherConfig(kind="chebyshev", weight=1.0, inner_iterations=solver.get("degree", 2),
                            lanczos_steps=solver.get("lanczos_steps", 10))
    else:
        sm = SmootherConfig(kind=solver["smoother"], weight=solver.get("weight", 0.5),
                            safeguard=solver.get("safeguard", 0.0))
    return sm
