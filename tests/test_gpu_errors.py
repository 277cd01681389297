"""Error functionals and the HDG projection on the GPU against
the oracle's compute_errors / hdg_project (postprocess.cpp:95-250), and the
README golden table (proj/README.md:78-82) reproduced by a study run entirely
on the device: device expansion + pattern, K1-K5, boundary data, CG solve,
postprocess and compute_errors."""
import numpy as np
import pytest
import torch

from gpu_util import np_, oracle_mesh
from oracle import core
from oracle_util import field, max_slice_relerr, vfield
from paper_1305_1489_b200.configs import CONFIGS, PAPER_SINE
from paper_1305_1489_b200.engine import Engine, HostMesh

pytestmark = pytest.mark.gpu


def _gpu_level(mesh, k, prob, tau=1.0):
    """study.cpp:10-43 on the GPU; returns everything compute_errors needs."""
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.expand(mesh.coordinates, mesh.elements, mesh.dirichlet, mesh.neumann)
    g = eng.geometry(dm, tau)
    cs = eng.build_condense(g, prob.kappa, prob.c, prob.f)
    pat = eng.pattern_device(dm)
    sysH = eng.assemble(dm, pat, cs)
    eng.neumann_load(dm, g, prob.q, b=sysH.b, alpha=-1.0)
    ub = eng.dirichlet_project(dm, prob.u)
    uhat, info = eng.solve_skeleton(dm, pat, sysH, ub, rtol=1e-14)
    ls = eng.recover(g, dm, cs, uhat)
    eng.set_postprocess_rule()
    ustar = eng.postprocess_star(g, prob.kappa, ls)
    eng.set_error_rule()
    return eng, dm, g, uhat, ls, ustar


def _oracle_ms(em, k, prob, tau=1.0):
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    taus = core.Stabilization(np.full((em.n_elements, 4), float(tau)))
    ms = core.build_element_matrices(em, t, field(prob.kappa), field(prob.c), field(prob.f), taus)
    return ms, taus


@pytest.mark.parametrize("k", [1, 2, 3])
def test_hdg_project(k):
    prob = CONFIGS["C2"].problem
    mesh = HostMesh.box(3, bc=prob.bc, perturb=0.1)
    em = oracle_mesh(mesh)
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    eng.set_error_rule()
    got = eng.hdg_project(g, prob.q, prob.u)
    ms, taus = _oracle_ms(em, k, prob)
    te = core.tables(k, 2 * k + 4, 2 * k + 4)
    want = core.hdg_project(em, ms, te, taus, vfield(prob.q), field(prob.u))
    for a, b in zip((got.qx, got.qy, got.qz, got.u), want):
        assert max_slice_relerr(np_(a), b.T) < 1e-10


@pytest.mark.parametrize("k,tau", [(1, 1.0), (2, 1.0), (3, 4.0)])
def test_compute_errors_match_oracle(k, tau):
    """Same discrete solution into both: the GPU functionals equal the oracle's."""
    prob = CONFIGS["C2"].problem
    mesh = HostMesh.box(3, bc=prob.bc, perturb=0.08)
    em = oracle_mesh(mesh)
    eng, dm, g, uhat, ls, ustar = _gpu_level(mesh, k, prob, tau)
    got = eng.compute_errors(dm, g, prob.q, prob.u, uhat, ls, ustar)
    ms, taus = _oracle_ms(em, k, prob, tau)
    want = core.compute_errors(em, ms, taus, field(prob.u), vfield(prob.q), k, np_(uhat),
                               np.asfortranarray(np_(ls.qx).T), np.asfortranarray(np_(ls.qy).T),
                               np.asfortranarray(np_(ls.qz).T), np.asfortranarray(np_(ls.u).T),
                               np.asfortranarray(np_(ustar).T))
    names = ("e_q", "e_u", "e_uhat", "eps_u", "eps_uhat", "e_star")
    for n, w in zip(names, want):
        assert abs(got[n] - w) <= 1e-9 * abs(w), (n, got[n], w)


def test_readme_golden_on_gpu():
    """proj/README.md:78-82 (paper-sine, k=1, tau=1, levels n = 2, 4, 8) from
    the all-GPU study; errors printed to 4 significant digits match."""
    want_eq = [3.9548e-02, 1.0547e-02, 2.6813e-03]
    want_eu = [6.4292e-02, 1.6866e-02, 4.2920e-03]
    for lev, n in enumerate([2, 4, 8]):
        mesh = HostMesh.box(n, bc="dirichlet_top_bottom")
        eng, dm, g, uhat, ls, ustar = _gpu_level(mesh, 1, PAPER_SINE)
        e = eng.compute_errors(dm, g, PAPER_SINE.q, PAPER_SINE.u, uhat, ls, ustar)
        assert float(f"{e['e_q']:.4e}") == want_eq[lev]
        assert float(f"{e['e_u']:.4e}") == want_eu[lev]
