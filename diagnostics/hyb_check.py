import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, ctypes as C
from oracle import topomg_oracle as O
from paper_2001_01655_b200 import problems as P
import paper_2001_01655_b200 as T
for dims in [(24,12,12),(48,24,24)]:
    w = P.config_4(dims=dims)
    g = O.make_grid(w.mesh.dims)
    E = O.simp_modulus(w.rho, 3, 1, 1e-9)
    K = O.assemble_stiffness(g, w.bc.fixed_dofs, E)
    sm = O.Smoother("chebyshev", 1.0, 2)
    hg = O.build_gmg(g, K, 999, sm, 1, 1)
    Kd = T.assemble_stiffness(w.mesh, w.bc, E)
    tsm = T.SmootherConfig(kind="chebyshev", weight=1.0, inner_iterations=2, lanczos_steps=10)
    B = T.rigid_body_modes(w.mesh, w.bc.fixed_dofs)
    dh = T.build_hybrid(w.mesh, Kd, B, 3, 999, tsm, 1, 1, beta=P.BETA, isolated="drop")
    dg = T.build_gmg(w.mesh, Kd, 999, tsm, 1, 1)
    x = np.random.default_rng(0).standard_normal(g.n_dofs)
    ref = hg.apply(x)
    r = lambda a: np.linalg.norm(a.cpu().numpy()-ref)/np.linalg.norm(ref)
    print(dims, [lv.size for lv in dh.levels], [lv.size for lv in dg.levels], "hyb %.2e gmg %.2e" % (r(dh.apply(x)), r(dg.apply(x))))
    print("  lmax hyb", [dh.level_lmax(k) for k in range(dh.n_levels-1)], "gmg", [dg.level_lmax(k) for k in range(dg.n_levels-1)],
          "oracle", [lv.smoother.bounds[1]/1.1 for lv in hg.levels[:-1]])
