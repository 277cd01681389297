"""Diagnostics: per-element C error of the structured condensation against the
oracle's LU path for a large constant kappa on part of the mesh, and the
recovery-cache factors against numpy (test infrastructure on the GPU box)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from gpu_util import np_, oracle_mesh  # noqa: E402
from oracle import core  # noqa: E402
from oracle_util import field  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
kap = sys.argv[2] if len(sys.argv) > 2 else "1 + 1e4*lt(0.5, x)"
c, f = "1 + x*y", "cos(x + y)"
mesh = HostMesh.box(2, bc="dirichlet_x")
em = oracle_mesh(mesh)
t = core.tables(k, 2 * k + 2, 2 * k + 2)
ms = core.build_element_matrices(em, t, field(kap), field(c), field(f), core.Stabilization(np.ones((em.n_elements, 4))))
lb = core.local_blocks(ms)
C, Cf = core.condense(lb, 1)
for jit in (True, False):
    eng = Engine(0)
    eng.set_degree(k)
    eng.set_jit(jit)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    cs = eng.build_condense(g, kap, c, f)
    Cg = np_(cs.C_slices())
    err = np.linalg.norm((Cg - C).reshape(len(C), -1), axis=1) / np.linalg.norm(C.reshape(len(C), -1), axis=1)
    print(f"jit={jit} k={k} kappa={kap}: worst elements", np.argsort(-err)[:6], err[np.argsort(-err)[:6]])
    # element matrices through the materialising kernel
    em_g = eng.element_matrices(g, kap, c, f)
    for name in ("Mkinv", "Mc"):
        got = np_(em_g[name]) if isinstance(em_g, dict) else None
        if got is not None:
            want = ms.get(name)
            e2 = np.max(np.linalg.norm((got - want).reshape(len(want), -1), axis=1) /
                        np.linalg.norm(want.reshape(len(want), -1), axis=1))
            print("  ", name, e2)
    eng.set_rescue_screen(2.0)
    cs2 = eng.build_condense(g, kap, c, f)
    Cg2 = np_(cs2.C_slices())
    err2 = np.linalg.norm((Cg2 - C).reshape(len(C), -1), axis=1) / np.linalg.norm(C.reshape(len(C), -1), axis=1)
    print("  rescue path worst", err2.max(), "rescued", eng.rescued_elements())
    # factors vs numpy structured algebra on the worst element
    K = int(np.argmax(err))
    d3 = (k + 1) * (k + 2) * (k + 3) // 6
    A1 = lb.A1[K]
    M = A1[:d3, :d3]
    F = np_(cs.factors.view(dm.nelt, -1))[K]
    ns = d3 * (d3 + 1) // 2
    def unpack(v):
        out = np.zeros((d3, d3))
        p = 0
        for j in range(d3):
            for i in range(j, d3):
                out[i, j] = out[j, i] = v[p]
                p += 1
        return out
    Mi = unpack(F[:ns])
    Cb = A1[3 * d3:, :3 * d3]
    D = A1[3 * d3:, 3 * d3:]
    Mi_ref = np.linalg.inv(M)
    Mbi = np.kron(np.eye(3), Mi_ref)
    S = D + Cb @ Mbi @ Cb.T
    E = lb.A3[K][:, :3 * d3]
    tDP = lb.A3[K][:, 3 * d3:]
    V = Cb @ Mbi @ E.T + tDP.T
    m = 4 * ((k + 1) * (k + 2) // 2)
    Vs = F[ns:ns + d3 * m].reshape(m, d3).T
    Vs_ref = np.linalg.solve(S, V)
    print("  element", K, "Mi err", np.linalg.norm(Mi - Mi_ref) / np.linalg.norm(Mi_ref),
          "Vs err", np.linalg.norm(Vs - Vs_ref) / np.linalg.norm(Vs_ref), "cond S", np.linalg.cond(S))
