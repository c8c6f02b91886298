"""Structured Q4/Hex8 meshes and the device stiffness operator.

Mirrors the reference's mesh module interface (reference mesh.py): ``build_mesh``,
``StructuredMesh``, ``BoundaryConditions``, ``element_stiffness``,
``assemble_stiffness``, ``rigid_body_modes``.  The difference is what
``assemble_stiffness`` returns: instead of a scipy CSR matrix it returns a
``StiffnessOperator`` that lives on the B200 and is applied matrix-free
(element moduli + the unit element matrix), with the same symmetric Dirichlet
elimination (unit diagonal) as mesh.py:313.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._dev import as_dev, empty_dev, ptr, stream_ptr

DEFAULT_NU = 0.3


@dataclass(frozen=True)
class StructuredMesh:
    """Uniform Q4/Hex8 grid; nodes lexicographic with x fastest (mesh.py:15)."""

    dims: tuple
    element_size: tuple

    def __post_init__(self):
        if len(self.dims) not in (2, 3):
            raise ValueError("mesh must be 2D or 3D, got dims=%r" % (self.dims,))
        if len(self.dims) != len(self.element_size):
            raise ValueError("dims and element_size length mismatch")
        if any(d < 1 for d in self.dims):
            raise ValueError("all dims must be >= 1")
        if any(h <= 0 for h in self.element_size):
            raise ValueError("all element sizes must be > 0")
        object.__setattr__(self, "dims", tuple(int(d) for d in self.dims))
        object.__setattr__(self, "element_size", tuple(float(h) for h in self.element_size))

    ndim = property(lambda self: len(self.dims))
    dofs_per_node = property(lambda self: len(self.dims))
    node_dims = property(lambda self: tuple(d + 1 for d in self.dims))
    node_count = property(lambda self: int(np.prod(self.node_dims)))
    element_count = property(lambda self: int(np.prod(self.dims)))
    total_dofs = property(lambda self: self.node_count * self.dofs_per_node)

    def node_index(self, *ijk):
        nd = self.node_dims
        if self.ndim == 2:
            return ijk[0] + nd[0] * ijk[1]
        return ijk[0] + nd[0] * (ijk[1] + nd[1] * ijk[2])

    def node_coordinates(self):
        grids = np.meshgrid(*[np.arange(n) * h for n, h in zip(self.node_dims, self.element_size)],
                            indexing="ij")
        return np.column_stack([g.reshape(-1, order="F") for g in grids])

    def element_nodes(self):
        ijk = [g.reshape(-1, order="F") for g in
               np.meshgrid(*[np.arange(d) for d in self.dims], indexing="ij")]
        quad = [(0, 0), (1, 0), (1, 1), (0, 1)]
        if self.ndim == 2:
            return np.column_stack([self.node_index(ijk[0] + a, ijk[1] + b) for a, b in quad])
        return np.column_stack([self.node_index(ijk[0] + a, ijk[1] + b, ijk[2] + c)
                                for c in (0, 1) for a, b in quad])

    def element_dofs(self):
        conn = self.element_nodes()
        dpn = self.dofs_per_node
        return (dpn * conn[:, :, None] + np.arange(dpn)).reshape(conn.shape[0], -1).astype(np.int64)

    def element_centroids(self):
        grids = np.meshgrid(*[(np.arange(d) + 0.5) * h for d, h in zip(self.dims, self.element_size)],
                            indexing="ij")
        return np.column_stack([g.reshape(-1, order="F") for g in grids])


@dataclass
class BoundaryConditions:
    """Fixed dofs plus nodal loads; loads zeroed on fixed dofs (mesh.py:121)."""

    fixed_dofs: np.ndarray
    load_vector: np.ndarray

    def __post_init__(self):
        self.fixed_dofs = np.unique(np.asarray(self.fixed_dofs, dtype=np.int64))
        self.load_vector = np.asarray(self.load_vector, dtype=float).copy()
        if self.fixed_dofs.size and self.fixed_dofs[-1] >= self.load_vector.size:
            raise ValueError("fixed dof index out of range")
        self.load_vector[self.fixed_dofs] = 0.0

    @property
    def free_mask(self):
        m = np.ones(self.load_vector.size, dtype=bool)
        m[self.fixed_dofs] = False
        return m


def build_mesh(dims, element_size=None):
    if element_size is None:
        element_size = [1.0] * len(dims)
    return StructuredMesh(tuple(dims), tuple(element_size))


def element_stiffness(mesh, E=1.0, nu=DEFAULT_NU):
    """Q4/Hex8 element matrix by 2-point Gauss quadrature (mesh.py:254), computed
    by the library's native host code."""
    nd = mesh.dofs_per_node * 2 ** mesh.ndim
    out = np.empty((nd, nd))
    _lib.check(_lib.load().tmg_element_stiffness(C.byref(_lib.mesh_desc(mesh)), float(E), float(nu),
                                                 out.ctypes.data))
    return out


class StiffnessOperator:
    """K(rho) on the device: ``K @ x`` (torch fp64 CUDA tensors), ``diagonal()``,
    ``shape``.  Owns a copy of the element moduli."""

    def __init__(self, mesh, bc, element_moduli, nu=DEFAULT_NU, stream=None):
        E = as_dev(element_moduli)
        if E.numel() != mesh.element_count:
            raise ValueError("element_moduli must have one entry per element")
        fixed = np.zeros(0, np.int64) if bc is None else np.ascontiguousarray(bc.fixed_dofs, np.int64)
        h = C.c_void_p()
        _lib.check(_lib.load().tmg_operator_create(
            C.byref(_lib.mesh_desc(mesh)), ptr(E), fixed.ctypes.data if fixed.size else None,
            int(fixed.size), float(nu), stream_ptr(stream), C.byref(h)))
        self._h = h
        self.mesh = mesh
        self.bc = bc
        self.nu = nu
        self.element_moduli = E
        n = mesh.total_dofs
        self.shape = (n, n)

    @property
    def handle(self):
        return self._h

    def matvec(self, x, out=None, stream=None):
        x = as_dev(x)
        if x.numel() != self.shape[0]:
            raise ValueError("dimension mismatch")
        out = empty_dev(self.shape[0]) if out is None else out
        _lib.check(_lib.load().tmg_operator_apply(self._h, ptr(x), ptr(out), stream_ptr(stream)))
        return out

    __matmul__ = matvec

    def diagonal(self):
        out = empty_dev(self.shape[0])
        _lib.check(_lib.load().tmg_operator_diagonal(self._h, ptr(out), stream_ptr(None)))
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.tmg_operator_destroy(h)
            self._h = None


def assemble_stiffness(mesh, bc, element_moduli, nu=DEFAULT_NU):
    """Device K(E) with Dirichlet elimination (mesh.py:327); bc=None keeps it singular."""
    moduli = element_moduli
    if isinstance(moduli, np.ndarray) or not hasattr(moduli, "is_cuda"):
        moduli = np.asarray(moduli, dtype=float)
        if moduli.shape != (mesh.element_count,):
            raise ValueError("element_moduli must have one entry per element")
        if np.any(moduli <= 0):
            raise ValueError("element moduli must be positive")
    return StiffnessOperator(mesh, bc, moduli, nu)


def rigid_body_modes(mesh, fixed_dofs=None):
    """Rigid-body candidates about the centroid (mesh.py:418), host array: this is
    hierarchy *input* data (the near-nullspace), not part of the device path."""
    X = mesh.node_coordinates()
    X = X - X.mean(axis=0)
    n, dpn = mesh.node_count, mesh.dofs_per_node
    if mesh.ndim == 2:
        B = np.zeros((2 * n, 3))
        B[0::2, 0] = B[1::2, 1] = 1.0
        B[0::2, 2], B[1::2, 2] = -X[:, 1], X[:, 0]
    else:
        B = np.zeros((3 * n, 6))
        for c in range(3):
            B[c::3, c] = 1.0
        B[0::3, 3], B[1::3, 3] = -X[:, 1], X[:, 0]
        B[1::3, 4], B[2::3, 4] = -X[:, 2], X[:, 1]
        B[0::3, 5], B[2::3, 5] = X[:, 2], -X[:, 0]
    if fixed_dofs is not None:
        B[np.asarray(fixed_dofs, dtype=np.int64)] = 0.0
    return B
