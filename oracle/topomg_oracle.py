"""CPU oracle for the MG-PCG hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy/scipy restatement of the reference algorithms
(`/root/reference/pkg/src/topomg/*.py`) for the path the B200 framework
accelerates: element stiffness, stiffness assembly with symmetric Dirichlet
elimination, geometric / smoothed-aggregation / hybrid multigrid hierarchies,
the V-cycle with its smoothers, the Krylov drivers and the compliance
sensitivity.  It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it.
The product path (``paper_2001_01655_b200``) never imports this file.

Parity pin: every function here is checked against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/topomg`` in the build container and writes
``tests/golden/reference_golden.npz``); see ``tests/test_oracle_golden.py``.

Extensions that the reference does not have (needed by BASELINE.json's
``north_star``) are marked EXTENSION and follow the same conventions:
preconditioned CG (the reference's krylov module says a CG extension is
possible, krylov.py design note), a Jacobi-preconditioned Chebyshev smoother
with a Lanczos eigenvalue bound, a level cap for geometric hierarchies, and a
configurable strength threshold for SA-AMG.
"""

from __future__ import annotations

import dataclasses
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

NU_DEFAULT = 0.3
BETA_DEFAULT = 0.003  # multigrid.py:22


# ---------------------------------------------------------------------------
# structured mesh (reference mesh.py:15-117)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Grid:
    """Uniform Q4/Hex8 grid, lexicographic nodes with x fastest (mesh.py:15)."""

    dims: tuple
    h: tuple

    @property
    def ndim(self):
        return len(self.dims)

    @property
    def dpn(self):
        return len(self.dims)

    @property
    def node_dims(self):
        return tuple(d + 1 for d in self.dims)

    @property
    def n_nodes(self):
        return int(np.prod(self.node_dims))

    @property
    def n_elems(self):
        return int(np.prod(self.dims))

    @property
    def n_dofs(self):
        return self.n_nodes * self.dpn

    def node_id(self, *ijk):  # mesh.py:65
        nd = self.node_dims
        if self.ndim == 2:
            return ijk[0] + nd[0] * ijk[1]
        return ijk[0] + nd[0] * (ijk[1] + nd[1] * ijk[2])

    def coords(self):  # mesh.py:58
        axes = [np.arange(n) * hh for n, hh in zip(self.node_dims, self.h)]
        mesh = np.meshgrid(*axes, indexing="ij")
        return np.column_stack([m.reshape(-1, order="F") for m in mesh])

    def connectivity(self):  # mesh.py:73 (counter-clockwise local order)
        idx = np.meshgrid(*[np.arange(d) for d in self.dims], indexing="ij")
        idx = [a.reshape(-1, order="F") for a in idx]
        if self.ndim == 2:
            i, j = idx
            corners = [(0, 0), (1, 0), (1, 1), (0, 1)]
            return np.column_stack([self.node_id(i + a, j + b) for a, b in corners])
        i, j, k = idx
        corners = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
                   (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
        return np.column_stack([self.node_id(i + a, j + b, k + c) for a, b, c in corners])

    def edofs(self):  # mesh.py:104 -- local dof = local_node*dpn + component
        conn = self.connectivity()
        dpn = self.dpn
        return (dpn * conn[:, :, None] + np.arange(dpn)[None, None, :]).reshape(conn.shape[0], -1)


def make_grid(dims, h=None):
    dims = tuple(int(d) for d in dims)
    if len(dims) not in (2, 3):
        raise ValueError("2D or 3D only")
    h = tuple(float(x) for x in (h if h is not None else [1.0] * len(dims)))
    if len(h) != len(dims):
        raise ValueError("dims/h mismatch")
    return Grid(dims, h)


# ---------------------------------------------------------------------------
# element matrices (mesh.py:162-267)
# ---------------------------------------------------------------------------

def _dshape(ndim, xi):
    """Natural-coordinate shape-function gradients (mesh.py:167)."""
    if ndim == 2:
        s, t = xi
        return 0.25 * np.array([[-(1 - t), (1 - t), (1 + t), -(1 + t)],
                                [-(1 - s), -(1 + s), (1 + s), (1 - s)]])
    s, t, u = xi
    ss = np.array([-1, 1, 1, -1, -1, 1, 1, -1], float)
    tt = np.array([-1, -1, 1, 1, -1, -1, 1, 1], float)
    uu = np.array([-1, -1, -1, -1, 1, 1, 1, 1], float)
    return 0.125 * np.array([ss * (1 + tt * t) * (1 + uu * u),
                             tt * (1 + ss * s) * (1 + uu * u),
                             uu * (1 + ss * s) * (1 + tt * t)])


def constitutive(ndim, E, nu):
    """Plane stress (2D, unit thickness) or isotropic 3D (mesh.py:191)."""
    if ndim == 2:
        return E / (1 - nu * nu) * np.array([[1, nu, 0], [nu, 1, 0], [0, 0, (1 - nu) / 2]])
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[range(3), range(3)] += 2 * mu
    D[3:, 3:] = np.eye(3) * mu
    return D


def strain_matrix(ndim, g):
    """B from physical gradients g (ndim, nodes) (mesh.py:208)."""
    nn = g.shape[1]
    if ndim == 2:
        B = np.zeros((3, 2 * nn))
        B[0, 0::2] = g[0]; B[1, 1::2] = g[1]
        B[2, 0::2] = g[1]; B[2, 1::2] = g[0]
        return B
    B = np.zeros((6, 3 * nn))
    B[0, 0::3] = g[0]; B[1, 1::3] = g[1]; B[2, 2::3] = g[2]
    B[3, 0::3] = g[1]; B[3, 1::3] = g[0]
    B[4, 1::3] = g[2]; B[4, 2::3] = g[1]
    B[5, 0::3] = g[2]; B[5, 2::3] = g[0]
    return B


def gauss_rule(grid):
    """(weight*detJ, physical gradient) per 2-point Gauss point (mesh.py:231)."""
    h = np.asarray(grid.h)
    jac = h / 2.0
    gp = np.array([-1.0, 1.0]) / np.sqrt(3.0)
    pts = np.array(np.meshgrid(*([gp] * grid.ndim), indexing="ij")).reshape(grid.ndim, -1).T
    return [(float(np.prod(jac)), _dshape(grid.ndim, p) / jac[:, None]) for p in pts]


def element_stiffness(grid, E=1.0, nu=NU_DEFAULT):
    """KE by 2x2(x2) Gauss quadrature, symmetrised (mesh.py:254)."""
    if not 0 <= nu < 0.5:
        raise ValueError("nu must be in [0, 0.5)")
    if E <= 0:
        raise ValueError("E must be positive")
    D = constitutive(grid.ndim, E, nu)
    n = grid.dpn * 2 ** grid.ndim
    ke = np.zeros((n, n))
    for w, g in gauss_rule(grid):
        B = strain_matrix(grid.ndim, g)
        ke += w * B.T @ D @ B
    return 0.5 * (ke + ke.T)


# ---------------------------------------------------------------------------
# assembly and boundary conditions (mesh.py:301-366)
# ---------------------------------------------------------------------------

def scatter(grid, blocks):
    ed = grid.edofs()
    m = ed.shape[1]
    r = np.repeat(ed, m, axis=1).ravel()
    c = np.tile(ed, (1, m)).ravel()
    K = sp.csr_matrix((blocks.ravel(), (r, c)), shape=(grid.n_dofs, grid.n_dofs))
    K.sum_duplicates()
    return K


def dirichlet(K, fixed):
    """Z K Z + I_fixed: zero fixed rows/cols, unit diagonal (mesh.py:313)."""
    n = K.shape[0]
    keep = np.ones(n)
    keep[fixed] = 0.0
    Z = sp.diags(keep)
    out = (Z @ K @ Z).tocsr() + sp.diags(1.0 - keep)
    out = out.tocsr()
    out.sum_duplicates()
    return out


def assemble_stiffness(grid, fixed, moduli, nu=NU_DEFAULT):
    """Global K(E) with Dirichlet elimination; fixed=None keeps it singular (mesh.py:327)."""
    moduli = np.asarray(moduli, float)
    if moduli.shape != (grid.n_elems,):
        raise ValueError("one modulus per element")
    if np.any(moduli <= 0):
        raise ValueError("moduli must be positive")
    ke = element_stiffness(grid, 1.0, nu)
    K = scatter(grid, moduli[:, None, None] * ke[None])
    return K if fixed is None else dirichlet(K, np.asarray(fixed, np.int64))


def rigid_body_modes(grid, fixed=None):
    """Translations + rotations about the centroid (mesh.py:418)."""
    X = grid.coords()
    X = X - X.mean(axis=0)
    n = grid.n_nodes
    if grid.ndim == 2:
        B = np.zeros((2 * n, 3))
        B[0::2, 0] = 1; B[1::2, 1] = 1
        B[0::2, 2] = -X[:, 1]; B[1::2, 2] = X[:, 0]
    else:
        B = np.zeros((3 * n, 6))
        for c in range(3):
            B[c::3, c] = 1
        B[0::3, 3] = -X[:, 1]; B[1::3, 3] = X[:, 0]
        B[1::3, 4] = -X[:, 2]; B[2::3, 4] = X[:, 1]
        B[0::3, 5] = X[:, 2]; B[2::3, 5] = -X[:, 0]
    if fixed is not None:
        B[np.asarray(fixed, np.int64)] = 0.0
    return B


def density_filter(grid, radius=1.5):
    """Row-normalised hat filter, radius in element units (mesh.py:369)."""
    if radius <= 0:
        raise ValueError("radius must be positive")
    reach = max(int(np.ceil(radius - 1e-12)) - 1, 0)
    rng = np.arange(-reach, reach + 1)
    offs = np.array(np.meshgrid(*([rng] * grid.ndim), indexing="ij")).reshape(grid.ndim, -1).T
    dist = np.sqrt((offs.astype(float) ** 2).sum(axis=1))
    sel = dist < radius
    offs, wts = offs[sel], radius - dist[sel]
    dims = np.array(grid.dims)
    idx = np.column_stack([a.reshape(-1, order="F") for a in
                           np.meshgrid(*[np.arange(d) for d in grid.dims], indexing="ij")])
    stride = np.cumprod([1] + list(grid.dims[:-1]))
    R, C, V = [], [], []
    for o, w in zip(offs, wts):
        nb = idx + o
        ok = np.all((nb >= 0) & (nb < dims), axis=1)
        R.append(idx[ok] @ stride); C.append(nb[ok] @ stride); V.append(np.full(ok.sum(), w))
    S = sp.csr_matrix((np.concatenate(V), (np.concatenate(R), np.concatenate(C))),
                      shape=(grid.n_elems, grid.n_elems))
    S = sp.diags(1.0 / np.asarray(S.sum(axis=1)).ravel()) @ S
    return S.tocsr()


# ---------------------------------------------------------------------------
# material law (material.py:8-50)
# ---------------------------------------------------------------------------

def simp_modulus(rho, penal, e0=1.0, emin=1e-10 * 1.0):
    rho = np.asarray(rho, float)
    if np.any((rho < 0) | (rho > 1)):
        raise ValueError("rho must lie in [0, 1]")
    return emin + (e0 - emin) * rho ** penal


def simp_derivative(rho, penal, e0=1.0, emin=1e-10):
    rho = np.asarray(rho, float)
    if penal == 1.0:
        return np.full_like(rho, e0 - emin)
    return penal * (e0 - emin) * rho ** (penal - 1.0)


# ---------------------------------------------------------------------------
# smoothers (multigrid.py:29-193) + EXTENSION: Jacobi-Chebyshev
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Smoother:
    kind: str = "weighted_jacobi"   # weighted_jacobi | block_jacobi | chebyshev | sor_chebyshev | sor_gmres
    weight: float = 0.5
    inner_iterations: int = 2       # Chebyshev degree
    block_size: int = 2
    lanczos_steps: int = 10         # EXTENSION (chebyshev)
    seed: int = 0                   # EXTENSION (chebyshev start vector)
    safeguard: float = 0.0          # EXTENSION: >0 caps the Jacobi weight at safeguard/lambda_hat

    def __post_init__(self):
        if not 0 < self.weight <= 1:
            raise ValueError("smoother weight must be in (0, 1]")
        if self.inner_iterations < 1:
            raise ValueError("inner_iterations must be >= 1")


def splitmix_uniform(n, seed=0):
    """EXTENSION: deterministic uniform(-1,1) start vector shared with the GPU.

    x_i = splitmix64(seed * 0x9E3779B97F4A7C15 + i + 1); value = (x >> 11) * 2^-53 * 2 - 1.
    """
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
             + np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def lanczos_max_eig(A, dinv, steps=10, seed=0):
    """EXTENSION: largest Ritz value of D^-1/2 A D^-1/2 after `steps` Lanczos steps."""
    ds = np.sqrt(dinv)
    v = splitmix_uniform(A.shape[0], seed)
    v = v / np.linalg.norm(v)
    vprev = np.zeros_like(v)
    alphas, betas = [], []
    beta = 0.0
    for _ in range(steps):
        w = ds * (A @ (ds * v))
        a = float(w @ v)
        w = w - a * v - beta * vprev
        beta = float(np.linalg.norm(w))
        alphas.append(a)
        if beta <= 1e-300:
            break
        betas.append(beta)
        vprev, v = v, w / beta
    m = len(alphas)
    T = np.diag(alphas) + np.diag(betas[:m - 1], 1) + np.diag(betas[:m - 1], -1)
    return float(np.linalg.eigvalsh(T)[-1])


class JacobiSweeps:
    """x += w D^-1 (b - A x) (multigrid.py:48)."""

    def __init__(self, A, cfg):
        d = A.diagonal()
        if np.any(d == 0):
            raise ValueError("zero diagonal entry; operator not smoothable")
        self.A, self.dinv, self.w = A, 1.0 / d, cfg.weight
        self.lmax_estimate = None
        if cfg.safeguard > 0:
            # EXTENSION: keep w*lambda_max(D^-1 A) below `safeguard` (< 2) so the
            # symmetric V-cycle stays SPD on Galerkin levels where it would not.
            self.lmax_estimate = lanczos_max_eig(A, self.dinv, cfg.lanczos_steps, cfg.seed)
            self.w = min(cfg.weight, cfg.safeguard / self.lmax_estimate)

    def apply(self, x, b, passes):
        for _ in range(passes):
            x = x + self.w * (self.dinv * (b - self.A @ x))
        return x


class BlockJacobiSweeps:
    """Nodal-block weighted Jacobi (multigrid.py:64)."""

    def __init__(self, A, cfg):
        bs = cfg.block_size
        n = A.shape[0]
        if n % bs:
            raise ValueError("matrix size not divisible by block size")
        nb = n // bs
        blk = np.zeros((nb, bs, bs))
        for a in range(bs):
            for b in range(bs):
                rows = np.arange(nb) * bs + a
                cols = np.arange(nb) * bs + b
                blk[:, a, b] = np.asarray(A[rows, cols]).ravel()
        if np.any(np.abs(np.linalg.det(blk)) < 1e-300):
            raise ValueError("singular nodal block in block Jacobi smoother")
        self.A, self.binv, self.bs, self.w = A, np.linalg.inv(blk), bs, cfg.weight

    def apply(self, x, b, passes):
        for _ in range(passes):
            r = (b - self.A @ x).reshape(-1, self.bs)
            x = x + self.w * np.einsum("nab,nb->na", self.binv, r).ravel()
        return x


class JacobiChebyshevSweeps:
    """EXTENSION: degree-k Chebyshev on D^-1 A, same recurrence as the reference's
    SOR-Chebyshev (multigrid.py:131) with the SOR solve replaced by D^-1 and the
    power-method bound replaced by a Lanczos bound; interval [0.1, 1.1]*lambda."""

    def __init__(self, A, cfg):
        d = A.diagonal()
        if np.any(d == 0):
            raise ValueError("zero diagonal entry; operator not smoothable")
        self.A, self.dinv, self.degree = A, 1.0 / d, cfg.inner_iterations
        self.lmax_estimate = lanczos_max_eig(A, self.dinv, cfg.lanczos_steps, cfg.seed)
        self.bounds = (0.1 * self.lmax_estimate, 1.1 * self.lmax_estimate)

    def apply(self, x, b, passes):
        lo, hi = self.bounds
        theta, delta = (hi + lo) / 2.0, (hi - lo) / 2.0
        for _ in range(passes):
            r = b - self.A @ x
            p = None
            alpha = 0.0
            for i in range(self.degree):
                z = self.dinv * r
                if i == 0:
                    p = z.copy()
                    alpha = 1.0 / theta
                else:
                    beta = (delta * alpha / 2.0) ** 2
                    alpha = 1.0 / (theta - beta / alpha)
                    p = z + beta * p
                x = x + alpha * p
                r = r - alpha * (self.A @ p)
        return x


class SorSolve:
    """One forward SOR (Gauss-Seidel, omega = 1) sweep as a preconditioner solve:
    z = tril(A)^-1 v (multigrid.py:97-106)."""

    def __init__(self, A):
        self.L = sp.tril(A, format="csr")
        if np.any(self.L.diagonal() == 0):
            raise ValueError("zero diagonal; SOR sweep undefined")

    def solve(self, v):
        return spla.spsolve_triangular(self.L, np.asarray(v, float), lower=True)


class SorChebyshevSweeps:
    """Fixed-degree Chebyshev polynomial in the SOR-preconditioned operator
    (multigrid.py:109-150): bounds [0.1, 1.1] * lambda, lambda from 10 power
    steps on tril(A)^-1 A from numpy default_rng(seed).standard_normal(n)."""

    def __init__(self, A, cfg, seed=0):
        self.A, self.sor, self.degree = A, SorSolve(A), cfg.inner_iterations
        v = np.random.default_rng(seed).standard_normal(A.shape[0])
        lam = 1.0
        for _ in range(10):
            v /= np.linalg.norm(v)
            w = self.sor.solve(A @ v)
            lam = float(np.linalg.norm(w))
            v = w
        self.lmax_estimate = lam
        self.bounds = (0.1 * lam, 1.1 * lam)

    def apply(self, x, b, passes):
        lo, hi = self.bounds
        d, c = (hi + lo) / 2.0, (hi - lo) / 2.0
        for _ in range(passes):
            r = b - self.A @ x
            alpha = 0.0
            p = None
            for i in range(self.degree):
                z = self.sor.solve(r)
                if i == 0:
                    p = z.copy()
                    alpha = 1.0 / d
                else:
                    beta = (c * alpha / 2.0) ** 2
                    alpha = 1.0 / (d - beta / alpha)
                    p = z + beta * p
                x = x + alpha * p
                r = r - alpha * (self.A @ p)
        return x


class SorGmresSweeps:
    """inner_iterations FGMRES steps right-preconditioned by one SOR sweep, per
    pass (multigrid.py:153-170: rtol 1e-14, max_iterations = restart = steps)."""

    def __init__(self, A, cfg):
        self.A, self.sor, self.steps = A, SorSolve(A), cfg.inner_iterations

    def apply(self, x, b, passes):
        for _ in range(passes):
            x, _ = gmres(self.A, b, x, self.sor.solve, rtol=1e-14, max_iterations=self.steps,
                         restart=self.steps, flexible=True)
        return x


SMOOTHERS = {"weighted_jacobi": JacobiSweeps, "block_jacobi": BlockJacobiSweeps,
             "chebyshev": JacobiChebyshevSweeps, "sor_chebyshev": SorChebyshevSweeps,
             "sor_gmres": SorGmresSweeps}


def make_smoother(cfg, A, block_size=None):
    if cfg.kind not in SMOOTHERS:
        raise ValueError("unknown smoother kind %r" % cfg.kind)
    if block_size is not None and cfg.kind == "block_jacobi" and block_size != cfg.block_size:
        cfg = dataclasses.replace(cfg, block_size=block_size)
    return SMOOTHERS[cfg.kind](A, cfg)


# ---------------------------------------------------------------------------
# hierarchy + V-cycle (multigrid.py:200-265)
# ---------------------------------------------------------------------------

@dataclass
class Level:
    A: sp.csr_matrix
    P: sp.csr_matrix | None
    provenance: str
    smoother: object = None
    aggregates: np.ndarray | None = None     # SA levels: node -> aggregate id
    strength: sp.csr_matrix | None = None    # SA levels: strength adjacency
    tentative: sp.csr_matrix | None = None   # SA levels: T
    omega: float | None = None               # SA levels: prolongation smoothing weight


@dataclass
class Hierarchy:
    levels: list
    coarse_solve: object
    n_pre: int = 1
    n_post: int = 1
    flags: list = field(default_factory=list)
    smoother_cfg: Smoother | None = None

    @property
    def n_levels(self):
        return len(self.levels)

    @property
    def n_geometric(self):
        return sum(lv.provenance == "geometric" for lv in self.levels[:-1])

    def vcycle(self, b, k=0):
        """Alg. 1 with zero initial guess (multigrid.py:231)."""
        if not 0 <= k < len(self.levels):
            raise IndexError("level index out of range")
        lv = self.levels[k]
        if lv.P is None:
            return self.coarse_solve(b)
        x = lv.smoother.apply(np.zeros_like(b), b, self.n_pre)
        r = b - lv.A @ x
        x = x + lv.P @ self.vcycle(lv.P.T @ r, k + 1)
        return lv.smoother.apply(x, b, self.n_post)

    def apply(self, b):
        return self.vcycle(b, 0)

    def summary(self):
        return [{"size": int(lv.A.shape[0]), "nonzeros": int(lv.A.nnz),
                 "provenance": lv.provenance} for lv in self.levels]


def finalize(levels, n_pre, n_post, flags, cfg):
    lu = spla.splu(levels[-1].A.tocsc())
    return Hierarchy(levels, lu.solve, n_pre, n_post, flags, cfg)


def galerkin(A, P):
    Ac = (P.T @ A @ P).tocsr()
    Ac.sum_duplicates()
    return Ac


# -- geometric (multigrid.py:272-336) --

def coarsen_dims(dims):
    return tuple(max(1, -(-d // 2)) for d in dims)


def gmg_plan(dims, dpn, coarse_max_dofs, max_levels=None):
    """Element dims per level; EXTENSION: optional max_levels cap."""
    plan = [tuple(dims)]
    while True:
        cur = plan[-1]
        if dpn * int(np.prod([d + 1 for d in cur])) <= coarse_max_dofs or all(d <= 1 for d in cur):
            break
        if max_levels is not None and len(plan) >= max_levels:
            break
        plan.append(coarsen_dims(cur))
    return plan


def hat_1d(n):
    """(n+1) x (ceil(n/2)+1) linear interpolation (multigrid.py:288)."""
    m = max(1, -(-n // 2))
    P = sp.lil_matrix((n + 1, m + 1))
    for i in range(n + 1):
        if i % 2 == 0:
            P[i, i // 2] = 1.0
        else:
            P[i, (i - 1) // 2] = 0.5
            P[i, (i + 1) // 2] = 0.5
    return P.tocsr()


def geometric_prolongation(dims, dpn):
    """Kronecker product of 1D hats, x fastest, times I_dpn (multigrid.py:304)."""
    parts = [hat_1d(d) if d > 1 else sp.identity(d + 1, format="csr") for d in dims]
    Pn = parts[0]
    for p in parts[1:]:
        Pn = sp.kron(p, Pn, format="csr")
    return sp.kron(Pn, sp.identity(dpn), format="csr")


def build_gmg(grid, K, coarse_max_dofs, smoother=None, n_pre=1, n_post=1, max_levels=None):
    smoother = smoother or Smoother()
    plan = gmg_plan(grid.dims, grid.dpn, coarse_max_dofs, max_levels)
    flags = [] if len(plan) > 1 else ["no_coarsening_possible"]
    levels, A = [], sp.csr_matrix(K)
    for dims in plan[:-1]:
        P = geometric_prolongation(dims, grid.dpn)
        levels.append(Level(A, P, "geometric", make_smoother(smoother, A, grid.dpn)))
        A = galerkin(A, P)
    levels.append(Level(A, None, "geometric"))
    if A.shape[0] > coarse_max_dofs and max_levels is None:
        flags.append("coarse_bound_not_reached")
    return finalize(levels, n_pre, n_post, flags, smoother)


# -- smoothed aggregation (multigrid.py:343-566) --

def strength_graph(K, beta=BETA_DEFAULT, block_size=1):
    """Edge (I,J) iff ||K_IJ||_F^2 > beta*||K_II||_F*||K_JJ||_F (multigrid.py:355)."""
    K = sp.csr_matrix(K)
    if K.shape[0] % block_size:
        raise ValueError("matrix size not divisible by block size")
    nb = K.shape[0] // block_size
    sq = K.multiply(K)
    if block_size > 1:
        R = sp.kron(sp.identity(nb), np.ones((1, block_size)), format="csr")
        M = (R @ sq @ R.T).tocsr()
    else:
        M = sq.tocsr()
    dg = M.diagonal()
    if np.any(dg == 0):
        raise ValueError("zero diagonal block; input looks unassembled or singular")
    C = M.tocoo()
    keep = (C.row != C.col) & (C.data > beta * np.sqrt(dg[C.row] * dg[C.col]))
    return sp.csr_matrix((np.ones(keep.sum()), (C.row[keep], C.col[keep])), shape=(nb, nb))


def aggregate(adj, isolated="merge"):
    """Greedy root pass, neighbour absorption, isolated/forced fallbacks (multigrid.py:380).

    EXTENSION isolated="drop": nodes without strong connections stay unaggregated
    (id -1, zero rows of T -- PyAMG standard_aggregation semantics) instead of
    becoming singletons that _merge_small_aggregates folds into ONE aggregate."""
    n = adj.shape[0]
    ptr, ind = adj.indptr, adj.indices
    agg = -np.ones(n, np.int64)
    count = 0
    for i in range(n):
        if agg[i] >= 0:
            continue
        nb = ind[ptr[i]:ptr[i + 1]]
        if nb.size and np.all(agg[nb] < 0):
            agg[i] = count
            agg[nb] = count
            count += 1
    for i in range(n):
        if agg[i] >= 0:
            continue
        nb = ind[ptr[i]:ptr[i + 1]]
        hit = nb[agg[nb] >= 0]
        if hit.size:
            agg[i] = agg[hit[0]]
    flags = []
    lone = np.flatnonzero(agg < 0)
    if count == 0 or count + lone.size >= n:
        return np.arange(n) // 2, ["forced_pairwise_aggregation"]
    if lone.size:
        if isolated == "merge":
            agg[lone] = count + np.arange(lone.size)
        flags.append("isolated_nodes")
    return agg, flags


def _renumber(agg):
    """np.unique(agg, return_inverse=True) over the aggregated nodes (-1 kept)."""
    out = agg.copy()
    m = agg >= 0
    out[m] = np.unique(agg[m], return_inverse=True)[1]
    return out


def merge_small(agg, adj, min_size):
    """Fold undersized aggregates into a strong neighbour, else an index neighbour
    (multigrid.py:427).  Unaggregated (-1) nodes are left alone (EXTENSION)."""
    size = np.bincount(agg[agg >= 0])
    small = np.flatnonzero(size < min_size)
    if small.size == 0:
        return agg
    agg, size = agg.copy(), size.copy()
    ptr, ind = adj.indptr, adj.indices
    for a in small:
        members = np.flatnonzero(agg == a)
        tgt = -1
        for i in members:
            for j in ind[ptr[i]:ptr[i + 1]]:
                if agg[j] != a and agg[j] >= 0 and size[agg[j]] >= min_size:
                    tgt = agg[j]
                    break
            if tgt >= 0:
                break
        if tgt >= 0:
            agg[members] = tgt
            size[tgt] += members.size
            size[a] = 0
    agg = _renumber(agg)
    while True:
        size = np.bincount(agg[agg >= 0])
        if size.size < 2:
            break
        small = np.flatnonzero(size < min_size)
        if small.size == 0:
            break
        a = small[0]
        agg[agg == a] = a - 1 if a > 0 else a + 1
        agg = _renumber(agg)
    return agg


def tentative(agg, B, block_size):
    """Per-aggregate thin QR of the candidate block (multigrid.py:471)."""
    B = np.asarray(B, float)
    nv = B.shape[1]
    na = int(agg.max()) + 1
    order = np.argsort(agg, kind="stable")
    cuts = np.searchsorted(agg[order], np.arange(na + 1))
    Bc = np.zeros((na * nv, nv))
    R_, C_, V_ = [], [], []
    for a in range(na):
        nodes = order[cuts[a]:cuts[a + 1]]
        dofs = (nodes[:, None] * block_size + np.arange(block_size)).ravel()
        if dofs.size < nv:
            raise ValueError("aggregate with %d dofs cannot carry %d candidates" % (dofs.size, nv))
        Q, R = np.linalg.qr(B[dofs])
        k = Q.shape[1]
        R_.append(np.repeat(dofs, k)); C_.append(np.tile(a * nv + np.arange(k), dofs.size))
        V_.append(Q.ravel())
        Bc[a * nv:a * nv + k] = R
    T = sp.csr_matrix((np.concatenate(V_), (np.concatenate(R_), np.concatenate(C_))),
                      shape=(B.shape[0], na * nv))
    return T, Bc


def spectral_radius(A, dinv=None, iterations=10, seed=0, v0=None):
    """Power method on D^-1 A from default_rng(seed).standard_normal (multigrid.py:504)."""
    if dinv is None:
        dinv = 1.0 / A.diagonal()
    v = np.random.default_rng(seed).standard_normal(A.shape[0]) if v0 is None else v0.copy()
    lam = 1.0
    for _ in range(iterations):
        v = v / np.linalg.norm(v)
        v = dinv * (A @ v)
        lam = float(np.linalg.norm(v))
    return max(lam, 1e-30)


def smooth_prolongation(A, T, seed=0):
    """P = T - (4/(3 rho)) D^-1 A T (multigrid.py:518). Returns (P, omega)."""
    dinv = 1.0 / A.diagonal()
    omega = 4.0 / (3.0 * spectral_radius(A, dinv, seed=seed))
    P = (T - sp.diags(omega * dinv) @ (A @ T)).tocsr()
    P.sum_duplicates()
    return P, omega


def sa_levels(A, B, coarse_max_dofs, smoother, block_size, flags, max_levels=30, seed=0,
              beta=BETA_DEFAULT, isolated="merge"):
    """multigrid.py:528; EXTENSION: beta parameter (reference fixes 0.003), isolated mode."""
    levels = []
    nv = B.shape[1]
    while A.shape[0] > coarse_max_dofs and len(levels) < max_levels:
        min_nodes = max(2, -(-nv // block_size))
        S = strength_graph(A, beta, block_size)
        agg, f = aggregate(S, isolated)
        flags.extend(f)
        agg = merge_small(agg, S, min_nodes)
        if (int(agg.max()) + 1) * nv >= A.shape[0]:
            flags.append("aggregation_stalled")
            break
        T, Bc = tentative(agg, B, block_size)
        P, omega = smooth_prolongation(A, T, seed)
        levels.append(Level(A, P, "algebraic", make_smoother(smoother, A, block_size),
                            aggregates=agg, strength=S, tentative=T, omega=omega))
        A = galerkin(A, P)
        B = Bc
        block_size = nv
    levels.append(Level(A, None, "algebraic"))
    return levels


def build_sa_amg(K, B, coarse_max_dofs, smoother=None, n_pre=1, n_post=1, seed=0,
                 beta=BETA_DEFAULT, isolated="merge"):
    smoother = smoother or Smoother()
    B = np.asarray(B, float)
    if B.ndim != 2 or B.shape[0] != K.shape[0]:
        raise ValueError("near_nullspace must be (ndofs, nvec)")
    bs = {3: 2, 6: 3}.get(B.shape[1], 1)
    flags = []
    levels = sa_levels(sp.csr_matrix(K), B, coarse_max_dofs, smoother, bs, flags, seed=seed,
                       beta=beta, isolated=isolated)
    return finalize(levels, n_pre, n_post, flags, smoother)


def jitter(B, rel, seed=7):
    """TEST-ONLY perturbation of SA candidates by rel (reproducibility floors: a
    rounding-level change of the setup input)."""
    B = np.asarray(B, float)
    if not rel:
        return B
    return B * (1.0 + rel * np.random.default_rng(seed).standard_normal(B.shape))


def build_hybrid(grid, K, B, n_geo, coarse_max_dofs, smoother=None, n_pre=1, n_post=1,
                 seed=0, beta=BETA_DEFAULT, isolated="merge", candidate_jitter=0.0):
    """Geometric on the finest n_geo levels, SA below (multigrid.py:573).
    candidate_jitter: test-only, see jitter()."""
    smoother = smoother or Smoother()
    if n_geo <= 0:
        return build_sa_amg(K, B, coarse_max_dofs, smoother, n_pre, n_post, seed, beta, isolated)
    flags, levels = [], []
    A = sp.csr_matrix(K)
    dims, h = grid.dims, grid.h
    for _ in range(n_geo):
        if all(d <= 1 for d in dims):
            flags.append("geometric_coarsening_exhausted")
            break
        if A.shape[0] <= coarse_max_dofs:
            break
        P = geometric_prolongation(dims, grid.dpn)
        levels.append(Level(A, P, "geometric", make_smoother(smoother, A, grid.dpn)))
        A = galerkin(A, P)
        dims = coarsen_dims(dims)
        h = tuple(2 * x for x in h)
    cgrid = Grid(dims, h)
    levels += sa_levels(A, jitter(rigid_body_modes(cgrid), candidate_jitter), coarse_max_dofs, smoother, cgrid.dpn,
                        flags, seed=seed, beta=beta, isolated=isolated)
    return finalize(levels, n_pre, n_post, flags, smoother)


# ---------------------------------------------------------------------------
# Krylov drivers (krylov.py) + EXTENSION: PCG
# ---------------------------------------------------------------------------

@dataclass
class Record:
    iterations: int = 0
    setup_time: float = 0.0
    solve_time: float = 0.0
    residual_history: list = field(default_factory=list)
    converged: bool = False


def _dot(x, y):
    return float(x @ y)


def pcg(A, b, x0=None, M=None, rtol=1e-8, max_iterations=1000, dot=None, observe=None):
    """EXTENSION: preconditioned CG under the reference's convergence contract.

    Tolerance relative to ||b|| (krylov.py:63).  Like the reference's restarted
    GMRES cycle (krylov.py:124-129), a cycle ends when the RECURSIVE residual
    meets the tolerance (or the iteration cap is hit); the TRUE residual
    ||b - A x|| then replaces the last history entry, and CG restarts from it when
    it misses the tolerance (residual replacement).  ``converged`` is the true
    residual test of krylov.py:128-129.

    ``dot``: alternative summation order of the dot products (reproducibility
    floors); ``observe(it, x)``: called after every iteration (fixture
    checkpoints)."""
    t0 = time.perf_counter()
    dot = dot or _dot
    b = np.asarray(b, float)
    x = np.zeros_like(b) if x0 is None else np.asarray(x0, float).copy()
    r = b - A @ x
    tol = rtol * np.sqrt(dot(b, b))
    rn = np.sqrt(dot(r, r))
    rec = Record(residual_history=[rn])
    it = 0
    while rn > tol and it < max_iterations:
        z = M(r) if M is not None else r.copy()
        p = z.copy()
        rz = dot(r, z)
        while True:
            q = A @ p
            alpha = rz / dot(p, q)
            x += alpha * p
            r -= alpha * q
            rn = np.sqrt(dot(r, r))
            it += 1
            rec.residual_history.append(rn)
            if observe is not None:
                observe(it, x)
            if rn <= tol or it >= max_iterations:
                break
            z = M(r) if M is not None else r.copy()
            rz_new = dot(r, z)
            p = z + (rz_new / rz) * p
            rz = rz_new
        r = b - A @ x                       # true residual (krylov.py:124-125)
        rn = np.sqrt(dot(r, r))
        rec.residual_history[-1] = rn
    rec.iterations = it
    rec.converged = bool(rn <= tol)
    rec.solve_time = time.perf_counter() - t0
    return x, rec


def gmres(A, b, x0=None, M=None, rtol=1e-7, max_iterations=1000, restart=200, flexible=False):
    """Right-preconditioned restarted (F)GMRES, MGS Arnoldi + Givens (krylov.py:48)."""
    t0 = time.perf_counter()
    M = M or (lambda v: v)
    b = np.asarray(b, float)
    x = np.zeros_like(b) if x0 is None else np.asarray(x0, float).copy()
    r = b - A @ x
    rec = Record(residual_history=[float(np.linalg.norm(r))])
    tol = rtol * float(np.linalg.norm(b))
    if rec.residual_history[0] <= tol:
        rec.converged = True
        rec.solve_time = time.perf_counter() - t0
        return x, rec
    done, broke = 0, False
    while done < max_iterations and not broke:
        beta = float(np.linalg.norm(r))
        if beta <= tol:
            break
        m = min(restart, max_iterations - done)
        V = np.empty((m + 1, b.size))
        Z = np.empty((m, b.size)) if flexible else None
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        used = 0
        for j in range(m):
            z = M(V[j])
            if flexible:
                Z[j] = z
            w = A @ z
            for i in range(j + 1):
                H[i, j] = float(V[i] @ w)
                w -= H[i, j] * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            bd = H[j + 1, j] < 1e-14
            if not bd:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / den if den else 1.0
            sn[j] = H[j + 1, j] / den if den else 0.0
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            done += 1
            used = j + 1
            rec.residual_history.append(abs(g[j + 1]))
            if abs(g[j + 1]) <= tol or bd or done >= max_iterations:
                broke = bd
                break
        if used:
            y = np.linalg.solve(np.triu(H[:used, :used]), g[:used])
            x = x + (Z[:used].T @ y if flexible else M(V[:used].T @ y))
        r = b - A @ x
        rec.residual_history[-1] = float(np.linalg.norm(r))
        if rec.residual_history[-1] <= tol:
            break
    rec.iterations = done
    rec.converged = float(np.linalg.norm(b - A @ x)) <= tol
    rec.solve_time = time.perf_counter() - t0
    return x, rec


# ---------------------------------------------------------------------------
# sensitivity (optimization.py:106-132)
# ---------------------------------------------------------------------------

def strain_energies(grid, u, ke=None):
    """u_e^T KE u_e with the unit-modulus KE (optimization.py:106)."""
    ke = element_stiffness(grid) if ke is None else ke
    ue = np.asarray(u)[grid.edofs()]
    return np.einsum("ei,ij,ej->e", ue, ke, ue)


def compliance_sensitivity(grid, f, u, rho, penal, e0=1.0, emin=1e-10, ke=None):
    """(f^T u, dc = -dE/drho * u_e^T KE u_e) (optimization.py:128-129)."""
    dc = -simp_derivative(rho, penal, e0, emin) * strain_energies(grid, u, ke)
    return float(np.asarray(f) @ np.asarray(u)), dc
