"""Connectivity of the seeded density fields of the BASELINE configs: solid
(rho = 1) connected components, whether any component joins the supports to
the loaded nodes (a load path), and the volume fraction.

    python tools/config_stats.py [configs...]
"""
import os
import sys

import numpy as np
from scipy import ndimage

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2001_01655_b200 import problems  # noqa: E402


def main(which):
    for c in which:
        w = problems.CONFIGS[c]()
        dims = w.mesh.dims
        rho = w.rho.reshape(dims[::-1]).transpose() if len(dims) == 3 else w.rho.reshape(dims[::-1]).T
        solid = rho > 0.5
        lab, n = ndimage.label(solid)
        # elements at x = 0 (supports) and the elements touching loaded nodes
        left = set(np.unique(lab[0][lab[0] > 0]).tolist())
        f = w.bc.load_vector
        dpn = w.mesh.ndim
        loaded = np.nonzero(np.abs(f.reshape(-1, dpn)).sum(1))[0]
        load_labels = set()
        for node in loaded:
            if dpn == 2:
                i, j = node % (dims[0] + 1), node // (dims[0] + 1)
                for ei in (i - 1, i):
                    for ej in (j - 1, j):
                        if 0 <= ei < dims[0] and 0 <= ej < dims[1] and lab[ei, ej] > 0:
                            load_labels.add(int(lab[ei, ej]))
            else:
                nx, ny = dims[0] + 1, dims[1] + 1
                i, j, k = node % nx, (node // nx) % ny, node // (nx * ny)
                for ei in (i - 1, i):
                    for ej in (j - 1, j):
                        for ek in (k - 1, k):
                            if (0 <= ei < dims[0] and 0 <= ej < dims[1] and 0 <= ek < dims[2]
                                    and lab[ei, ej, ek] > 0):
                                load_labels.add(int(lab[ei, ej, ek]))
        sizes = np.bincount(lab.ravel())[1:]
        print("config %d %s: volfrac %.3f, %d solid components (largest %.1f%% of solid), "
              "%d touch x=0, %d of %d loaded nodes touch solid, load path: %s"
              % (c, w.name, solid.mean(), n, 100.0 * sizes.max() / sizes.sum(), len(left),
                 sum(1 for _ in load_labels), len(loaded), bool(left & load_labels)), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4])
