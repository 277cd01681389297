"""Per-element check of K3 at C3 against the oracle on sampled elements:
the cached packed M^-1 and C (diagnostics for the k = 5 inverse): c3_inv_check.py [LIB]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_1305_1489_b200 import _lib as L  # noqa: E402

if len(sys.argv) > 1:
    L.LIB_PATH = os.path.abspath(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from gpu_util import oracle_condense, submesh, np_  # noqa: E402
from paper_1305_1489_b200.configs import CONFIGS  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh  # noqa: E402

cfg = CONFIGS["C3"]
prob = cfg.problem
mesh = HostMesh.box(cfg.n, bc=prob.bc, perturb=cfg.perturb, seed=cfg.seed)
eng = Engine(0)
eng.set_degree(cfg.k)
dm = eng.upload(mesh)
g = eng.geometry(dm, cfg.tau)
cs = eng.build_condense(g, prob.kappa, prob.c, prob.f)
nelt = dm.nelt
sel = np.unique(np.linspace(0, nelt - 1, 40).astype(int))
fb = mesh.facebyele
chosen, used = [], set()
for K in sel:
    if used.isdisjoint(fb[K]):
        chosen.append(K)
        used.update(fb[K])
sub = submesh(mesh, chosen)
_, _, lb, C, Cf = oracle_condense(sub, cfg.k, prob.kappa, prob.c, prob.f, cfg.tau)
A1 = np.asarray(lb.A1)
d3 = 56
F = np_(cs.factors.view(nelt, -1))
Cg = np_(cs.C_slices())
ns = d3 * (d3 + 1) // 2
for n, K in enumerate(chosen):
    A = A1[n]
    M = A[:d3, :d3]
    Mi = np.linalg.inv(M)
    pk = F[K, :ns]
    G = np.zeros((d3, d3))
    idx = 0
    for c in range(d3):
        for i in range(c, d3):
            G[i, c] = G[c, i] = pk[idx]
            idx += 1
    em = np.linalg.norm(G - Mi) / np.linalg.norm(Mi)
    ec = np.linalg.norm(Cg[K] - C[n]) / np.linalg.norm(C[n])
    D = A[3 * d3:, 3 * d3:]
    Cs = [A[3 * d3:, s * d3:(s + 1) * d3] for s in range(3)]
    S = D + sum(c @ Mi @ c.T for c in Cs)
    Af = np.asarray(lb.Af)
    fo = (Af[:, n] if Af.shape[0] == 4 * d3 else Af[n])[3 * d3:]
    fs_ref = np.linalg.solve(S, fo.reshape(-1))
    fs = F[K, ns + d3 * 84: ns + d3 * 84 + d3]
    ef = np.linalg.norm(fs - fs_ref) / np.linalg.norm(fs_ref)
    print(f"K {K}: Minv err {em:.1e}  C err {ec:.1e}  fs err {ef:.1e}  cond(S) {np.linalg.cond(S):.1e}")
