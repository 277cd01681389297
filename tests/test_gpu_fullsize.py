"""Every element of the bench configuration C2 (k = 3, 32^3 Kuhn box,
196,608 tets) and of C4 (k = 2, 48^3, upwind tau; C3 and C5 on request)
against the oracle's reference path, streamed over
16,384-element ranges of the full mesh (oracle.core.pipeline_range on all
host cores): C, Cf, and q, u recovered from the same lambda, within the
1e-10 contract; the pivot screen rescues nothing on this healthy mesh."""
import os

import numpy as np
import pytest
import torch

from gpu_util import TOL, np_, oracle_mesh
from oracle import core
from oracle_util import field
from paper_1305_1489_b200.configs import CONFIGS
from paper_1305_1489_b200.engine import Engine, HostMesh, dim2

pytestmark = pytest.mark.gpu


def _rel(got, want):
    got = got.reshape(got.shape[0], -1)
    want = want.reshape(want.shape[0], -1)
    return np.linalg.norm(got - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-300)


# C2 and C4 always; HDG_FULLSIZE_CONFIGS=C3,C5 adds the other BASELINE meshes (about a minute of oracle
# time each on 16 cores; profiles/r02f_fullsize_parity.txt holds a run of all of them)
_CONFIGS = ["C2", "C4"] + [c for c in os.environ.get("HDG_FULLSIZE_CONFIGS", "").split(",") if c in ("C3", "C5")]


@pytest.mark.parametrize("cfg_name", _CONFIGS)
def test_every_element_matches_oracle(cfg_name):
    cfg = CONFIGS[cfg_name]
    prob = cfg.problem
    k = cfg.k
    mesh = HostMesh.box(cfg.n, bc=prob.bc, perturb=cfg.perturb, seed=cfg.seed)
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, cfg.tau)
    tau_dev = eng.upwind_tau(g, cfg.upwind_beta) if cfg.upwind_beta else None   # C4: tau = 1 + |beta . nu|
    if tau_dev is not None:
        g = eng.geometry(dm, tau_dev)
    cs = eng.build_condense(g, prob.kappa, prob.c, prob.f)
    assert eng.rescued_elements() == 0
    d2 = dim2(k)
    uhat = torch.sin(torch.arange(dm.nfc * d2, dtype=torch.float64, device="cuda") * 0.013)
    ls = eng.recover(g, dm, cs, uhat)
    torch.cuda.synchronize()
    em = oracle_mesh(mesh)
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    tau = core.Stabilization(np.asfortranarray(np_(tau_dev).T) if tau_dev is not None
                             else np.full((em.n_elements, 4), float(cfg.tau)))
    kap, c, f = field(prob.kappa), field(prob.c), field(prob.f)
    lam = np.asfortranarray(core.gather_traces(em, d2, np_(uhat)))
    nelt, chunk = dm.nelt, 16384
    worst = {"C": 0.0, "Cf": 0.0, "qx": 0.0, "qy": 0.0, "qz": 0.0, "u": 0.0}
    Cg = cs.C_slices()
    Cfg = cs.Cf_cols()
    for k0 in range(0, nelt, chunk):
        k1 = min(nelt, k0 + chunk)
        C, Cf, qx, qy, qz, u = core.pipeline_range(em, t, kap, c, f, tau, np.asfortranarray(lam[:, k0:k1]),
                                                   k0, k1, os.cpu_count() or 1)
        got = {"C": np_(Cg[k0:k1]), "Cf": np_(Cfg[k0:k1]), "qx": np_(ls.qx[k0:k1]), "qy": np_(ls.qy[k0:k1]),
               "qz": np_(ls.qz[k0:k1]), "u": np_(ls.u[k0:k1])}
        want = {"C": C, "Cf": Cf.T, "qx": qx.T, "qy": qy.T, "qz": qz.T, "u": u.T}
        for name in worst:
            worst[name] = max(worst[name], float(_rel(got[name], want[name]).max()))
    print(f"{cfg_name}: max relative error over all {nelt} elements:", worst)
    assert all(v < TOL for v in worst.values()), worst
