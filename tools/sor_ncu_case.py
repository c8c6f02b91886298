import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2001_01655_b200 as T
from paper_2001_01655_b200 import _lib, problems
L=_lib.load(); w=problems.CONFIGS[1]()
law=T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
K=T.StiffnessOperator(w.mesh, w.bc, law.modulus(torch.as_tensor(w.rho, device="cuda")))
h=T.build_gmg(w.mesh, K, 1, T.SmootherConfig(kind="sor_gmres"), 1, 1, max_levels=5)
ms=C.c_double()
_lib.check(L.tmg_hierarchy_time_smoother(h.handle, 3, 2, C.byref(ms), None))
print(ms.value)
