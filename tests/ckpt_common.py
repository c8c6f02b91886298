"""Shared helpers of the fixed-iteration checkpoint fixtures (test infrastructure).

A full-size iterate (0.6-5.4 M doubles) is too large for a fixture, so every
checkpoint stores the compliance f.x_k, ||x_k|| and x_k projected on NPROJ
seeded Gaussian vectors.  For Gaussian W, ||W(x - y)|| / ||W y|| estimates
||x - y|| / ||y|| (relative spread ~ 1/sqrt(2 NPROJ)), so a device iterate is
compared with the oracle's without storing either.

Used by tests/golden/make_checkpoints.py (writes the fixtures on the CPU) and
tests/test_gpu_configs.py (checks the device against them)."""

import numpy as np

NPROJ = 16
PROJ_SEED = 20010165
# iterations at which the iterates are pinned, per config (capped by each run)
CHECKPOINTS = (10, 50, 200, 1000, 2000, 3000)


def project(x, nproj=NPROJ, seed=PROJ_SEED):
    """W x for W = default_rng(seed + i).standard_normal(n), row by row (no n x
    nproj matrix in memory)."""
    x = np.asarray(x, dtype=float)
    return np.array([np.random.default_rng(seed + i).standard_normal(x.size) @ x for i in range(nproj)])


def proj_rel(px, py):
    """||W x - W y|| / ||W y||: estimate of ||x - y|| / ||y||."""
    return float(np.linalg.norm(np.asarray(px) - np.asarray(py)) / np.linalg.norm(py))


def block_dot(x, y, nblk=296):
    """The GPU's two-level reduction order (296 block partials, then their sum)."""
    return float(sum(np.add.reduce(c) for c in np.array_split(x * y, nblk)))


class Reordered:
    """K @ x with every row summed in the REVERSE column order (the columns of K
    and the entries of x reversed, indices re-sorted): the same operator at
    another fp64 summation order.  (K^T @ x would not do: K is exactly symmetric,
    so CSR rows of K^T hold the same entries in the same order.)"""

    def __init__(self, K):
        import scipy.sparse as sp
        K = sp.csr_matrix(K)
        n = K.shape[1]
        self.Kr = sp.csr_matrix((K.data.copy(), n - 1 - K.indices, K.indptr.copy()), shape=K.shape)
        self.Kr.sort_indices()
        self.shape = K.shape

    def __matmul__(self, x):
        return self.Kr @ np.ascontiguousarray(x[::-1])


def other_coarse_solve(h):
    """Replace an oracle hierarchy's coarsest SuperLU solve by dense Cholesky (LU
    of the transpose if the matrix is not numerically SPD): an equally
    backward-stable solver -- what the device's Cholesky-based coarse inverse is
    to the reference's splu (multigrid.py:256-258).  Returns the previous solve."""
    import scipy.linalg as sla
    A = h.levels[-1].A.toarray()
    old = h.coarse_solve
    try:
        cf = sla.cho_factor(A)
        h.coarse_solve = lambda b: sla.cho_solve(cf, b)
    except np.linalg.LinAlgError:
        lu = sla.lu_factor(A.T)
        h.coarse_solve = lambda b: sla.lu_solve(lu, b, trans=1)
    return old
