import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np
from oracle import topomg_oracle as O
import paper_2001_01655_b200 as T
from test_gpu_parity import cantilever, host, rel
mesh, g, bc, rho, E, K, Kref = cantilever((12, 6, 6), 7, void=True)
B = T.rigid_body_modes(mesh, bc.fixed_dofs)
h = T.build_sa_amg(K, B, 60, T.SmootherConfig(weight=0.6), 2, 2, beta=0.0064, isolated="drop")
ho = O.build_sa_amg(Kref, O.rigid_body_modes(g, bc.fixed_dofs), 60, O.Smoother(weight=0.6), 2, 2, beta=0.0064, isolated="drop")
print("levels", [lv.size for lv in h.levels], [lv.A.shape[0] for lv in ho.levels])
rng = np.random.default_rng(1)
for t in range(3):
    b = rng.standard_normal(g.n_dofs)
    print("vcycle rel diff", rel(host(h.apply(b)), ho.apply(b)))
kc = len(ho.levels) - 1
bc_ = rng.standard_normal(ho.levels[kc].A.shape[0])
print("coarse solve rel diff", rel(host(h.vcycle(bc_, kc)), ho.vcycle(bc_, kc)), "cond", np.linalg.cond(ho.levels[kc].A.toarray()))
for k in range(kc):
    x = rng.standard_normal(ho.levels[k].A.shape[0])
    print("level", k, "A rel diff", rel(host(h.level_apply(k, x)), ho.levels[k].A @ x))
u, rec = T.cg_solve(K, bc.load_vector, None, h, T.SolveConfig(rtol=1e-8, max_iterations=3000))
uo, reco = O.pcg(Kref, bc.load_vector, None, ho.apply, rtol=1e-8, max_iterations=3000)
print("iters", rec.iterations, reco.iterations)
print("gpu hist tail", np.array(rec.residual_history[-4:]) / rec.residual_history[0])
print("orc hist tail", np.array(reco.residual_history[-4:]) / reco.residual_history[0])
print("hist rel diff first 10", np.abs(np.array(rec.residual_history[:10]) - np.array(reco.residual_history[:10])) / np.array(reco.residual_history[:10]))
# degenerate aggregates: rank of the aggregate's candidate block below nvec
agg, _ = h.aggregates(0)
B0 = O.rigid_body_modes(g, bc.fixed_dofs)
bad = 0
for a in range(agg.max() + 1):
    nodes = np.where(agg == a)[0]
    rows = np.concatenate([3 * nodes + c for c in range(3)])
    if np.linalg.matrix_rank(B0[rows]) < 6:
        bad += 1
print("aggregates with rank-deficient candidate blocks:", bad, "of", agg.max() + 1)
