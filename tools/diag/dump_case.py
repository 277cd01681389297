"""Dump the GPU condensation of one small case (C, Cf, recovery cache) plus
the oracle's element matrices for offline analysis: dump_case.py k kappa out.npz"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from gpu_util import np_  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh  # noqa: E402

k, kap, out = int(sys.argv[1]), sys.argv[2], sys.argv[3]
c, f = "1 + x*y", "cos(x + y)"
mesh = HostMesh.box(2, bc="dirichlet_x")
eng = Engine(0)
eng.set_degree(k)
dm = eng.upload(mesh)
g = eng.geometry(dm, 1.0)
cs = eng.build_condense(g, kap, c, f)
em = eng.element_matrices(g, kap, c, f)
np.savez(out, C=np_(cs.C_slices()), Cf=np_(cs.Cf_cols()), F=np_(cs.factors.view(dm.nelt, -1)),
         **{"em_" + n: np_(t) for n, t in em.items()})
print("dumped", out)
