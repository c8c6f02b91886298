"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/reference_golden.npz.  The oracle (oracle/topomg_oracle.py)
is pinned against this file in tests/test_oracle_golden.py; the GPU path is then
checked against the oracle.
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from topomg import krylov, mesh, multigrid, optimization  # noqa: E402
from topomg.material import SimpLaw  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")


def cantilever(dims, seed, void=False):
    m = mesh.build_mesh(dims, [1.0] * len(dims))
    dpn = m.dofs_per_node
    ny = dims[1]
    if len(dims) == 2:
        left = [m.node_index(0, j) for j in range(ny + 1)]
    else:
        left = [m.node_index(0, j, k) for j in range(ny + 1) for k in range(dims[2] + 1)]
    fixed = np.array([dpn * n + c for n in left for c in range(dpn)])
    f = np.zeros(m.total_dofs)
    tip = m.node_index(*([dims[0]] + [d // 2 for d in dims[1:]]))
    f[dpn * tip + 1] = -1.0
    bc = mesh.BoundaryConditions(fixed, f)
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.05, 1.0, m.element_count)
    if void:
        rho = np.where(rng.uniform(size=m.element_count) < 0.3, 1e-3, 1.0)
    E = SimpLaw(penalty=3.0, e_min_ratio=1e-9).modulus(rho)
    K = mesh.assemble_stiffness(m, bc, E)
    return m, bc, rho, E, K


def dense(A):
    return A.toarray() if sp.issparse(A) else np.asarray(A)


def main():
    g = {}
    # element matrices
    for tag, dims, h in (("q4", (1, 1), (1.0, 1.0)), ("q4h", (1, 1), (0.5, 0.25)),
                         ("hex8", (1, 1, 1), (1.0, 1.0, 1.0)),
                         ("hex8h", (1, 1, 1), (0.5, 0.5, 0.25))):
        m = mesh.build_mesh(dims, h)
        g["ke_" + tag] = mesh.element_stiffness(m, 1.0, 0.3)
    # assembly + BCs + rigid body modes + filter
    m, bc, rho, E, K = cantilever((6, 4), 1)
    g["asm_E"], g["asm_fixed"], g["asm_K"] = E, bc.fixed_dofs, dense(K)
    g["rbm_2d"] = mesh.rigid_body_modes(m, bc.fixed_dofs)
    m3 = mesh.build_mesh((3, 2, 2), (1.0, 1.0, 1.0))
    g["rbm_3d"] = mesh.rigid_body_modes(m3)
    g["filter_5x5"] = dense(mesh.build_filter(mesh.build_mesh((5, 5)), 1.5).matrix)
    g["filter_3d"] = dense(mesh.build_filter(mesh.build_mesh((3, 3, 2)), 1.5).matrix)
    # geometric prolongations (even / odd / unit dims)
    for dims in ((4, 2), (5, 3), (6, 1), (4, 2, 2), (3, 2, 1)):
        key = "P_" + "x".join(map(str, dims))
        g[key] = dense(multigrid.geometric_prolongation(dims, len(dims)))
    # GMG hierarchy 2D (jacobi 0.6, 2/2) and V-cycle
    rng = np.random.default_rng(7)
    m, bc, rho, E, K = cantilever((16, 8), 2)
    sm = multigrid.SmootherConfig(kind="weighted_jacobi", weight=0.6)
    h = multigrid.build_gmg(m, K, 60, sm, n_pre=2, n_post=2)
    g["gmg2d_E"], g["gmg2d_fixed"] = E, bc.fixed_dofs
    g["gmg2d_sizes"] = np.array([lv.A.shape[0] for lv in h.levels])
    g["gmg2d_A1"] = dense(h.levels[1].A)
    b = rng.standard_normal(K.shape[0])
    g["gmg2d_b"], g["gmg2d_vc"] = b, h.apply(b)
    # GMRES with GMG preconditioner
    x, rec = krylov.gmres_solve(K, bc.load_vector, None, h.apply, krylov.SolveConfig(rtol=1e-8))
    g["gmg2d_f"], g["gmg2d_gmres_x"] = bc.load_vector, x
    g["gmg2d_gmres_hist"] = np.array(rec.residual_history)
    x, rec = krylov.fgmres_solve(K, bc.load_vector, None, h.apply,
                                 krylov.SolveConfig(method="fgmres", rtol=1e-8, restart=5))
    g["gmg2d_fgmres_x"], g["gmg2d_fgmres_hist"] = x, np.array(rec.residual_history)
    # block Jacobi GMG V-cycle
    hb = multigrid.build_gmg(m, K, 60, multigrid.SmootherConfig(kind="block_jacobi", weight=0.5))
    g["gmg2d_bj_vc"] = hb.apply(b)
    # GMG hierarchy 3D, odd dims
    m3, bc3, rho3, E3, K3 = cantilever((5, 3, 3), 3)
    h3 = multigrid.build_gmg(m3, K3, 50, multigrid.SmootherConfig(weight=0.6), 1, 1)
    g["gmg3d_E"], g["gmg3d_fixed"] = E3, bc3.fixed_dofs
    g["gmg3d_sizes"] = np.array([lv.A.shape[0] for lv in h3.levels])
    g["gmg3d_Alast"] = dense(h3.levels[-1].A)
    b3 = rng.standard_normal(K3.shape[0])
    g["gmg3d_b"], g["gmg3d_vc"] = b3, h3.apply(b3)
    # SA-AMG pieces (2D with voids, 3D)
    for tag, dims, seed in (("sa2d", (12, 8), 4), ("sa3d", (6, 4, 4), 5)):
        mm, bcc, rr, EE, KK = cantilever(dims, seed, void=True)
        bs = mm.dofs_per_node
        B = mesh.rigid_body_modes(mm, bcc.fixed_dofs)
        S = multigrid.strength_of_connection(KK, 0.08, bs)
        agg0, fl = multigrid.aggregate_nodes(S)
        agg = multigrid._merge_small_aggregates(agg0, S.adjacency, 2)
        T, Bc = multigrid.tentative_prolongation(agg, B, bs)
        P = multigrid.smoothed_prolongation(KK, T)
        g[tag + "_E"], g[tag + "_fixed"] = EE, bcc.fixed_dofs
        g[tag + "_S"] = dense(S.adjacency)
        g[tag + "_agg0"], g[tag + "_agg"] = agg0, agg
        g[tag + "_T"], g[tag + "_Bc"], g[tag + "_P"] = dense(T), Bc, dense(P)
        g[tag + "_rho"] = np.array(multigrid.estimate_spectral_radius(KK))
        ha = multigrid.build_sa_amg(KK, B, 40, multigrid.SmootherConfig(weight=0.6), 2, 2)
        g[tag + "_sizes"] = np.array([lv.A.shape[0] for lv in ha.levels])
        bb = rng.standard_normal(KK.shape[0])
        g[tag + "_b"], g[tag + "_vc"] = bb, ha.apply(bb)
    # default-beta hierarchy (0.003) for the 2D case
    mm, bcc, rr, EE, KK = cantilever((12, 8), 4, void=True)
    B = mesh.rigid_body_modes(mm, bcc.fixed_dofs)
    ha = multigrid.build_sa_amg(KK, B, 40)
    g["sa2d_default_sizes"] = np.array([lv.A.shape[0] for lv in ha.levels])
    g["sa2d_default_vc"] = ha.apply(g["sa2d_b"])
    # degenerate graph -> forced pairwise
    Sdeg = multigrid.strength_of_connection(sp.identity(8, format="csr") * 3.0, block_size=1)
    g["forced_agg"] = multigrid.aggregate_nodes(Sdeg)[0]
    # hybrid 3D
    m3, bc3, rho3, E3, K3 = cantilever((8, 4, 4), 6)
    B3 = mesh.rigid_body_modes(m3, bc3.fixed_dofs)
    hh = multigrid.build_hybrid(m3, K3, B3, 1, 60, multigrid.SmootherConfig(weight=0.6))
    g["hyb3d_E"], g["hyb3d_fixed"] = E3, bc3.fixed_dofs
    g["hyb3d_sizes"] = np.array([lv.A.shape[0] for lv in hh.levels])
    g["hyb3d_prov"] = np.array([lv.provenance == "geometric" for lv in hh.levels])
    b3 = rng.standard_normal(K3.shape[0])
    g["hyb3d_b"], g["hyb3d_vc"] = b3, hh.apply(b3)
    # sensitivities
    m, bc, rho, E, K = cantilever((6, 4), 8)
    u = rng.standard_normal(m.total_dofs)
    g["sens_rho"], g["sens_u"] = rho, u
    g["sens_ce"] = optimization.element_strain_energies(m, u)
    g["sens_dE"] = SimpLaw(penalty=3.0, e_min_ratio=1e-9).modulus_derivative(rho)
    m3 = mesh.build_mesh((3, 2, 2), (1.0, 1.0, 1.0))
    u3 = rng.standard_normal(m3.total_dofs)
    g["sens3_u"], g["sens3_ce"] = u3, optimization.element_strain_energies(m3, u3)
    # SOR smoothers (multigrid.py:97-176) and block Jacobi on SA levels; own rng so
    # the arrays above stay unchanged
    rs = np.random.default_rng(11)
    m, bc, rho, E, K = cantilever((16, 8), 2)
    bsor = rs.standard_normal(K.shape[0])
    g["sor2d_b"] = bsor
    for kind in ("sor_chebyshev", "sor_gmres"):
        hs = multigrid.build_gmg(m, K, 60, multigrid.SmootherConfig(kind=kind), 1, 1)
        g["sor2d_%s_vc" % kind] = hs.apply(bsor)
        if kind == "sor_chebyshev":
            g["sor2d_lmax"] = np.array([lv.smoother.lmax_estimate for lv in hs.levels[:-1]])
        one = multigrid.smooth(multigrid.SmootherConfig(kind=kind, inner_iterations=3), K,
                               np.zeros(K.shape[0]), bsor, passes=2)
        g["sor2d_%s_smooth" % kind] = one
    # FGMRES preconditioned by a sor_gmres V-cycle (reference test_krylov.py:67)
    hs = multigrid.build_gmg(m, K, 60, multigrid.SmootherConfig(kind="sor_gmres"))
    x, rec = krylov.fgmres_solve(K, bc.load_vector, None, hs.apply,
                                 krylov.SolveConfig(method="fgmres", rtol=1e-8))
    g["sor2d_fgmres_x"], g["sor2d_fgmres_hist"] = x, np.array(rec.residual_history)
    # SA (2D voids) with SOR smoothers and with block Jacobi (3x3 blocks below level 0)
    mm, bcc, rr, EE, KK = cantilever((12, 8), 4, void=True)
    B = mesh.rigid_body_modes(mm, bcc.fixed_dofs)
    bsa = rs.standard_normal(KK.shape[0])
    g["sorsa_b"] = bsa
    for kind in ("sor_chebyshev", "sor_gmres", "block_jacobi"):
        ha = multigrid.build_sa_amg(KK, B, 40, multigrid.SmootherConfig(kind=kind, weight=0.6), 1, 1)
        g["sorsa_%s_vc" % kind] = ha.apply(bsa)
    # 3D GMG with the SOR-Chebyshev smoother
    m3, bc3, rho3, E3, K3 = cantilever((5, 3, 3), 3)
    h3 = multigrid.build_gmg(m3, K3, 50, multigrid.SmootherConfig(kind="sor_chebyshev"), 1, 1)
    b3 = rs.standard_normal(K3.shape[0])
    g["sor3d_b"], g["sor3d_vc"] = b3, h3.apply(b3)
    g["sor3d_lmax"] = np.array([lv.smoother.lmax_estimate for lv in h3.levels[:-1]])
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, len(g), "arrays", os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
