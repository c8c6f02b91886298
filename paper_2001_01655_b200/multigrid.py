"""Multigrid hierarchies on the B200 (mirrors reference multigrid.py).

``build_gmg(mesh, K, coarse_max_dofs, smoother, n_pre, n_post)`` returns an
``MgHierarchy`` whose levels live on the device: level 0 is the matrix-free
stiffness operator, coarse levels are Galerkin 3^d-point block stencils
(P^T A P computed on the GPU), the coarsest level is inverted densely once.
``vcycle``/``apply`` run Alg. 1 (multigrid.py:231) with a zero initial guess.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._dev import as_dev, empty_dev, ptr, stream_ptr

SMOOTHER_KINDS = {"weighted_jacobi": 0, "block_jacobi": 1, "chebyshev": 2, "sor_chebyshev": 3, "sor_gmres": 4}
PROVENANCE = {0: "geometric", 1: "algebraic"}
DEFAULT_STRENGTH_BETA = 0.003  # multigrid.py:22


@dataclass(frozen=True)
class SmootherConfig:
    """multigrid.py:30; kinds weighted_jacobi | block_jacobi | sor_chebyshev |
    sor_gmres as the reference, plus 'chebyshev': the Jacobi-preconditioned
    Chebyshev extension (degree = inner_iterations, Lanczos bound over
    lanczos_steps)."""

    kind: str = "weighted_jacobi"
    weight: float = 0.5
    inner_iterations: int = 2
    block_size: int = 2
    lanczos_steps: int = 10
    seed: int = 0
    safeguard: float = 0.0  # weighted_jacobi: cap w at safeguard/lambda_hat per level (0 = off)

    def __post_init__(self):
        if not (0 < self.weight <= 1):
            raise ValueError("smoother weight must be in (0, 1]")
        if self.inner_iterations < 1:
            raise ValueError("inner_iterations must be >= 1")
        if self.safeguard and (self.kind != "weighted_jacobi" or not 0 < self.safeguard < 2):
            raise ValueError("safeguard applies to weighted_jacobi only and must be in (0, 2)")

    @property
    def stationary(self):
        """True if repeated application is a fixed linear operator (multigrid.py:43).
        The extension kind "chebyshev" (Jacobi-Chebyshev with fixed Lanczos-bound
        coefficients) is a fixed symmetric polynomial in D^-1 A, hence stationary;
        the reference's SOR-based kinds are not."""
        return self.kind in ("weighted_jacobi", "block_jacobi", "chebyshev")

    def desc(self, ndofs=0):
        """C-ABI descriptor.  sor_chebyshev carries its power-method start vector
        (multigrid.py:118-119: default_rng(0), the smoother is built with seed 0)
        for the finest level's ndofs; coarser levels use its prefix."""
        if self.kind not in SMOOTHER_KINDS:
            raise ValueError("unknown smoother kind %r" % self.kind)
        d = _lib.SmootherDesc()
        if self.kind == "sor_chebyshev":
            d._power_start = np.ascontiguousarray(np.random.default_rng(0).standard_normal(int(ndofs)))
            d.power_start = d._power_start.ctypes.data
        d.kind = SMOOTHER_KINDS[self.kind]
        d.weight = float(self.weight)
        d.inner_iterations = int(self.inner_iterations)
        d.lanczos_steps = int(self.lanczos_steps)
        d.seed = int(self.seed)
        d.safeguard = float(self.safeguard)
        return d


@dataclass
class LevelView:
    size: int
    nonzeros: int
    provenance: str
    storage: str


class MgHierarchy:
    """Device-resident hierarchy (multigrid.py:208)."""

    _STORAGE = {0: "matrix_free", 1: "stencil", 2: "bsr", 3: "dense_inverse"}

    def __init__(self, handle, K, smoother_config, n_pre, n_post, flags=()):
        self._h = handle
        self.K = K
        self.smoother_config = smoother_config
        self.n_pre = n_pre
        self.n_post = n_post
        self.flags = list(flags)

    @property
    def handle(self):
        return self._h

    @property
    def n_levels(self):
        return _lib.load().tmg_hierarchy_num_levels(self._h)

    @property
    def levels(self):
        out = []
        for k in range(self.n_levels):
            info = _lib.LevelInfo()
            _lib.check(_lib.load().tmg_hierarchy_level_info(self._h, k, C.byref(info)))
            out.append(LevelView(int(info.size), int(info.nonzeros), PROVENANCE[info.provenance],
                                 self._STORAGE[info.storage]))
        return out

    @property
    def n_geometric(self):
        return sum(1 for lv in self.levels[:-1] if lv.provenance == "geometric")

    @property
    def stationary(self):
        return self.smoother_config is None or self.smoother_config.stationary

    def vcycle(self, b, k=0, out=None, stream=None):
        if not (0 <= k < self.n_levels):
            raise IndexError("level index out of range")
        b = as_dev(b)
        out = empty_dev(b.numel()) if out is None else out
        _lib.check(_lib.load().tmg_hierarchy_vcycle(self._h, k, ptr(b), ptr(out), stream_ptr(stream)))
        return out

    def apply(self, b, out=None, stream=None):
        return self.vcycle(b, 0, out, stream)

    __call__ = apply

    def smooth(self, x, b, passes=1, k=0, stream=None):
        """`passes` passes of the level-k smoother on x (in place on a device
        copy, returned): the smoother's apply(x, b, passes) (multigrid.py:57)."""
        b = as_dev(b)
        x = as_dev(x).clone()
        _lib.check(_lib.load().tmg_hierarchy_smooth(self._h, int(k), ptr(b), ptr(x), int(passes), stream_ptr(stream)))
        return x

    def level_apply(self, k, x):
        x = as_dev(x)
        out = empty_dev(x.numel())
        _lib.check(_lib.load().tmg_hierarchy_level_apply(self._h, k, ptr(x), ptr(out), stream_ptr(None)))
        return out

    def level_lmax(self, k):
        v = C.c_double()
        _lib.check(_lib.load().tmg_hierarchy_level_lmax(self._h, k, C.byref(v), stream_ptr(None)))
        return v.value

    def summary(self):
        return [{"size": lv.size, "nonzeros": lv.nonzeros, "provenance": lv.provenance}
                for lv in self.levels]

    def device_flags(self):
        buf = C.create_string_buffer(4096)
        _lib.check(_lib.load().tmg_hierarchy_flags(self._h, buf, 4096))
        s = buf.value.decode()
        return s.split(",") if s else []

    # -- parity exports (host copies of device data; tests only) --------------
    def _export(self, k, what):
        dims = (C.c_int64 * 4)()
        L = _lib.load()
        _lib.check(L.tmg_hierarchy_export(self._h, k, what, dims, None, None, None, stream_ptr(None)))
        nr, nc, nnz, rc = (int(v) for v in dims)
        rowptr = np.zeros(nr + 1, np.int32)
        col = np.zeros(max(nnz, 1), np.int32)
        R, Cc = (rc // 1000, rc % 1000) if rc else (0, 0)
        val = np.zeros(max(nnz * R * Cc, 1))
        _lib.check(L.tmg_hierarchy_export(self._h, k, what, dims, rowptr.ctypes.data, col.ctypes.data,
                                          val.ctypes.data, stream_ptr(None)))
        return nr, nc, nnz, R, Cc, rowptr, col[:nnz], val

    def _bsr(self, k, what):
        import scipy.sparse as sp
        nr, nc, nnz, R, Cc, rowptr, col, val = self._export(k, what)
        return sp.bsr_matrix((val[:nnz * R * Cc].reshape(nnz, R, Cc), col, rowptr),
                             shape=(nr * R, nc * Cc)).tocsr()

    def level_matrix(self, k):
        return self._bsr(k, 0)

    def prolongation(self, k):
        return self._bsr(k, 1)

    def tentative(self, k):
        return self._bsr(k, 4)

    def strength(self, k):
        import scipy.sparse as sp
        nr, nc, nnz, R, Cc, rowptr, col, val = self._export(k, 2)
        return sp.csr_matrix((np.ones(nnz), col, rowptr), shape=(nr, nr))

    def aggregates(self, k):
        dims = (C.c_int64 * 4)()
        L = _lib.load()
        _lib.check(L.tmg_hierarchy_export(self._h, k, 3, dims, None, None, None, stream_ptr(None)))
        agg = np.zeros(int(dims[0]), np.int32)
        rho = np.zeros(1)
        _lib.check(L.tmg_hierarchy_export(self._h, k, 3, dims, None, agg.ctypes.data, rho.ctypes.data,
                                          stream_ptr(None)))
        return agg.astype(np.int64), float(rho[0])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.tmg_hierarchy_destroy(h)
            self._h = None


def _coarsen_dims(dims):
    return tuple(max(1, -(-d // 2)) for d in dims)


def gmg_level_dims(dims, dofs_per_node, coarse_max_dofs, max_levels=None):
    """Planned element dims per level (multigrid.py:276; + optional level cap)."""
    out = [tuple(dims)]
    while True:
        cur = out[-1]
        if dofs_per_node * int(np.prod([d + 1 for d in cur])) <= coarse_max_dofs or all(d <= 1 for d in cur):
            break
        if max_levels is not None and len(out) >= max_levels:
            break
        out.append(_coarsen_dims(cur))
    return out


def build_gmg(mesh, K, coarse_max_dofs, smoother=None, n_pre=1, n_post=1, max_levels=None, stream=None):
    """Geometric hierarchy with Galerkin coarse operators (multigrid.py:318)."""
    smoother = smoother or SmootherConfig()
    if smoother.kind not in SMOOTHER_KINDS:
        raise ValueError("unknown smoother kind %r" % smoother.kind)
    if getattr(K, "mesh", mesh) is not mesh and K.mesh != mesh:
        raise ValueError("K was assembled on a different mesh")
    plan = gmg_level_dims(mesh.dims, mesh.dofs_per_node, coarse_max_dofs, max_levels)
    flags = [] if len(plan) > 1 else ["no_coarsening_possible"]
    if max_levels is None and mesh.dofs_per_node * int(np.prod([d + 1 for d in plan[-1]])) > coarse_max_dofs:
        flags.append("coarse_bound_not_reached")
    h = C.c_void_p()
    _lib.check(_lib.load().tmg_gmg_build(K.handle, int(coarse_max_dofs), int(max_levels or 0),
                                         C.byref(smoother.desc(K.shape[0])), int(n_pre), int(n_post),
                                         stream_ptr(stream), C.byref(h)))
    return MgHierarchy(h, K, smoother, n_pre, n_post, flags)


class DeviceSmoother(MgHierarchy):
    """make_smoother(config, A) of multigrid.py:179 for the stiffness operator:
    the finest level's smoother on the device, ``apply(x, b, passes)`` like the
    reference's smoother classes; ``lmax_estimate`` for the Chebyshev kinds."""

    def apply(self, x, b, passes=1, stream=None):  # noqa: D401 - reference signature
        return self.smooth(x, b, passes, 0, stream)

    __call__ = apply

    @property
    def lmax_estimate(self):
        return self.level_lmax(0)


def make_smoother(config, K, block_size=None, stream=None):
    """multigrid.py:179 on the device; K is the StiffnessOperator.  block_jacobi
    uses nodal blocks (block_size = dofs per node)."""
    if config.kind not in SMOOTHER_KINDS:
        raise ValueError("unknown smoother kind %r" % config.kind)
    dpn = K.mesh.dofs_per_node
    if config.kind == "block_jacobi" and (block_size or config.block_size) != dpn:
        raise ValueError("block_jacobi on the device uses nodal blocks of %d dofs" % dpn)
    h = C.c_void_p()
    _lib.check(_lib.load().tmg_smoother_create(K.handle, C.byref(config.desc(K.shape[0])), stream_ptr(stream),
                                               C.byref(h)))
    return DeviceSmoother(h, K, config, 0, 0)


def smooth(config, K, x, b, passes=1):
    """multigrid.py:190: `passes` smoothing passes of the configured kind on K x = b."""
    return make_smoother(config, K).apply(x, b, passes)


def _start_vector(n, seed):
    """numpy default_rng(seed).standard_normal(n): the power-method start vector of
    estimate_spectral_radius (multigrid.py:508-509); host-side input data."""
    return np.ascontiguousarray(np.random.default_rng(seed).standard_normal(n))


def _host_or_device(a):
    """(array, pointer): CUDA tensors are passed through, everything else becomes a
    C-contiguous fp64 numpy array (the C ABI copies either kind)."""
    if hasattr(a, "is_cuda") and a.is_cuda:
        a = a.contiguous()
        return a, a.data_ptr()
    a = np.ascontiguousarray(np.asarray(a, dtype=float))
    return a, a.ctypes.data


def build_sa_amg(K, near_nullspace, coarse_max_dofs, smoother=None, n_pre=1, n_post=1, seed=0,
                 beta=DEFAULT_STRENGTH_BETA, stream=None, v0=None, isolated="merge"):
    """Smoothed-aggregation hierarchy built on the device (multigrid.py:555).
    EXTENSION: beta (the reference fixes 0.003); v0 overrides the power-method start
    vector default_rng(seed).standard_normal(n) (e.g. a device-resident copy);
    isolated="drop" leaves strength-isolated nodes unaggregated instead of folding
    them into one aggregate (reference: "merge", multigrid.py:418-423/457-467)."""
    smoother = smoother or SmootherConfig()
    if smoother.kind not in SMOOTHER_KINDS:
        raise ValueError("unknown smoother kind %r" % smoother.kind)
    B, pB = _host_or_device(near_nullspace)
    if B.ndim != 2 or B.shape[0] != K.shape[0]:
        raise ValueError("near_nullspace must be (ndofs, nvec)")
    v0, pv = _host_or_device(_start_vector(K.shape[0], seed) if v0 is None else v0)
    h = C.c_void_p()
    _lib.check(_lib.load().tmg_sa_amg_build(K.handle, pB, B.shape[1], int(coarse_max_dofs),
                                            float(beta), pv, C.byref(smoother.desc(K.shape[0])),
                                            int(n_pre), int(n_post), isolated_mode(isolated),
                                            stream_ptr(stream), C.byref(h)))
    H = MgHierarchy(h, K, smoother, n_pre, n_post)
    H.flags = H.device_flags()
    return H


def isolated_mode(isolated):
    """C-ABI code of the isolated-node policy ("merge" = reference, "drop")."""
    if isolated not in ("merge", "drop"):
        raise ValueError("isolated must be 'merge' or 'drop', got %r" % (isolated,))
    return 0 if isolated == "merge" else 1


def hybrid_plan(mesh, n_geo, coarse_max_dofs):
    """Geometric part of build_hybrid (multigrid.py:589-601): (dims, sizes, flags)."""
    dims, sizes, flags = mesh.dims, mesh.element_size, []
    ndof = mesh.total_dofs
    for _ in range(n_geo):
        if all(d <= 1 for d in dims):
            flags.append("geometric_coarsening_exhausted")
            break
        if ndof <= coarse_max_dofs:
            break
        dims = _coarsen_dims(dims)
        sizes = tuple(2 * h for h in sizes)
        ndof = mesh.dofs_per_node * int(np.prod([d + 1 for d in dims]))
    return dims, sizes, flags


def build_hybrid(mesh, K, near_nullspace, n_geo, coarse_max_dofs, smoother=None, n_pre=1, n_post=1,
                 seed=0, beta=DEFAULT_STRENGTH_BETA, stream=None, isolated="merge"):
    """Geometric transfers on the finest n_geo levels, SA below (multigrid.py:573)."""
    from .mesh import StructuredMesh, rigid_body_modes
    smoother = smoother or SmootherConfig()
    if n_geo <= 0:
        return build_sa_amg(K, near_nullspace, coarse_max_dofs, smoother, n_pre, n_post, seed, beta, stream,
                            isolated=isolated)
    dims, sizes, _ = hybrid_plan(mesh, n_geo, coarse_max_dofs)
    Bc = np.ascontiguousarray(rigid_body_modes(StructuredMesh(dims, sizes)))
    v0 = _start_vector(Bc.shape[0], seed)
    h = C.c_void_p()
    _lib.check(_lib.load().tmg_hybrid_build(K.handle, int(n_geo), Bc.ctypes.data, Bc.shape[0], Bc.shape[1],
                                            int(coarse_max_dofs), float(beta), v0.ctypes.data,
                                            C.byref(smoother.desc(K.shape[0])), int(n_pre), int(n_post),
                                            isolated_mode(isolated), stream_ptr(stream), C.byref(h)))
    H = MgHierarchy(h, K, smoother, n_pre, n_post)
    H.flags = H.device_flags()
    return H


# ---------------------------------------------------------------------------
# adaptive hybrid controller (host logic, multigrid.py:614-631)
# ---------------------------------------------------------------------------
@dataclass
class AdaptiveHybridController:
    """Demote one geometric level whenever a solve needs too many iterations."""

    n_geo_current: int
    min_geo: int = 2
    iteration_threshold: int = 200

    def __post_init__(self):
        if self.n_geo_current < self.min_geo:
            raise ValueError("n_geo_current below the geometric floor")


def adapt_after_solve(ctrl, last_iterations):
    """Return 'rebuild' (and decrement n_geo) or 'keep' per the >threshold rule."""
    if last_iterations > ctrl.iteration_threshold and ctrl.n_geo_current > ctrl.min_geo:
        ctrl.n_geo_current -= 1
        return "rebuild"
    return "keep"
