"""Generate the committed golden fixtures (tests/golden/*.npz) from the CPU
oracle (pinned against the reference's KATs and README table, see
tests/test_oracle_kats.py). Run from the repo root:
    python tests/golden/make_golden.py
Each fixture holds a small seeded problem (perturbed 2^3 Kuhn box, Dirichlet
x = 0, 1 / Neumann elsewhere, C2-style variable coefficients) and the oracle's
outputs for its first elements: condensed C and Cf, recovered q and u for a
seeded skeleton vector, and the P_{k+1} postprocess u*."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import core  # noqa: E402
from oracle_util import field  # noqa: E402
from paper_1305_1489_b200.engine import HostMesh  # noqa: E402

KAP = "1 + 0.5*sin(2*pi*x)*cos(2*pi*y)"
CC = "1 + x*y*z"
FF = "exp(x + y)*sin(pi*z)"
NKEEP = 6  # elements kept per fixture


def make(k: int) -> dict:
    mesh = HostMesh.box(2, bc="dirichlet_x", perturb=0.1, seed=1305)
    em = core.expand(mesh.coordinates, mesh.elements, mesh.dirichlet, mesh.neumann)
    qd = 2 * k + 2
    t = core.tables(k, qd, qd)
    tau = core.Stabilization(np.full((em.n_elements, 4), 1.0))
    ms = core.build_element_matrices(em, t, field(KAP), field(CC), field(FF), tau)
    lb = core.local_blocks(ms)
    C, Cf = core.condense(lb, 1)
    d2 = (k + 1) * (k + 2) // 2
    uhat = np.random.default_rng(1305 + k).standard_normal(em.n_faces * d2)
    qx, qy, qz, u = core.local_recover(lb, core.gather_traces(em, d2, uhat), 1)
    t1 = core.tables(k + 1, 2 * (k + 1) + 2, qd)
    ustar = core.postprocess_star(em, t1, field(KAP), qx, qy, qz, u)
    return dict(k=k, kappa=KAP, c=CC, f=FF, coords=mesh.coordinates, elements=mesh.elements,
                dirichlet=mesh.dirichlet, neumann=mesh.neumann, faces=mesh.faces, facebyele=mesh.facebyele, facetype=mesh.facetype, uhat=uhat,
                C=C[:NKEEP], Cf=Cf[:, :NKEEP].T.copy(), qx=qx[:, :NKEEP].T.copy(), qy=qy[:, :NKEEP].T.copy(),
                qz=qz[:, :NKEEP].T.copy(), u=u[:, :NKEEP].T.copy(), ustar=ustar[:, :NKEEP].T.copy())


if __name__ == "__main__":
    for k in (1, 2, 3):
        np.savez_compressed(os.path.join(HERE, f"golden_k{k}.npz"), **make(k))
        print("wrote", f"golden_k{k}.npz")
