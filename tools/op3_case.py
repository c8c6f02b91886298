"""Config-4 level-0 operator kernels in isolation (timing / ncu target).

    python tools/op3_case.py [--reps 20]

Applies K(rho) of BASELINE config 4 (192x96x96 Hex8, 5.45 M dofs) through the
public API (K @ x -> k_apply<3>) and times it with CUDA events."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--config", type=int, default=4)
    a = p.parse_args()
    import numpy as np
    import torch

    import paper_2001_01655_b200 as T
    from paper_2001_01655_b200 import problems
    w = problems.CONFIGS[a.config]()
    law = T.SimpLaw(penalty=problems.PENAL, e_min_ratio=problems.EMIN)
    K = T.StiffnessOperator(w.mesh, w.bc, law.modulus(torch.as_tensor(w.rho, device="cuda")))
    x = torch.as_tensor(np.random.default_rng(0).standard_normal(w.ndof), device="cuda")
    y = K @ x
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        y = K @ x
    e1.record()
    torch.cuda.synchronize()
    print("k_apply<3> config %d: %.2f us per launch" % (a.config, 1e3 * e0.elapsed_time(e1) / a.reps))


if __name__ == "__main__":
    main()
