"""Structural invariants of the reference's acceptance suite on the CUDA path
(proj/tests/acceptance.cpp:243-409, criterion 7; tests/test_local_solver.cpp:
64-94): the flux identity between K3's (C, Cf) and K5's recovered (q, u), the
single-valuedness of the numerical flux on interior faces after a GPU solve,
mean preservation of the postprocess, and -- at BASELINE's full C2 size, where
the oracle is too slow to re-solve everything -- the size-independent
properties of the path (symmetry of C, linearity of the recovery in lambda,
mean preservation, the face-ordered scatter against a checksum of the
element contributions)."""
import numpy as np
import pytest
import torch

from gpu_util import gpu_pipeline, np_, oracle_condense, oracle_mesh
from oracle import core
from paper_1305_1489_b200.configs import CONFIGS, PAPER_SINE
from paper_1305_1489_b200.engine import Engine, HostMesh, dim2, dim3

pytestmark = pytest.mark.gpu

KAP = "2 + sin(x)*sin(y)*sin(z)"
CC = "1 + 0.5*(x*x + y*y + z*z)"
FF = "cos(x + 2*y - z)"


def _flux_moments(lb, ls, lam, K):
    """-A3 v + tauDD uhat for element K: the moments of the numerical flux
    q.n + tau (u - uhat) against the face bases (acceptance.cpp:318-327)."""
    v = np.concatenate([np_(ls.qx[K]), np_(ls.qy[K]), np_(ls.qz[K]), np_(ls.u[K])])
    return -lb.A3[K] @ v + lb.tauDD[K] @ lam


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_flux_identity(k):
    """-A3 v + tauDD uhat = C uhat - Cf on random traces (<= 1e-10,
    acceptance.cpp:310-331): C, Cf from K3, v from K5, A3 and tauDD from the
    oracle's local_blocks."""
    n = 2 if k < 4 else 1
    mesh = HostMesh.box(n, bc="dirichlet_x", perturb=0.1, seed=5)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    d2 = dim2(k)
    rng = np.random.default_rng(12345)
    uhat = rng.uniform(-0.5, 0.5, dm.nfc * d2)
    ls = eng.recover(g, dm, cs, torch.from_numpy(uhat).cuda())
    _, _, lb, _, _ = oracle_condense(em, k, KAP, CC, FF, 1.0)
    lam = core.gather_traces(em, d2, uhat)
    C, Cf = np_(cs.C_slices()), np_(cs.Cf_cols())
    worst = 0.0
    for K in range(em.n_elements):
        lhs = _flux_moments(lb, ls, lam[:, K], K)
        rhs = C[K] @ lam[:, K] - Cf[K]
        worst = max(worst, float(np.max(np.abs(lhs - rhs))))
    assert worst < 1e-10


@pytest.mark.parametrize("k", [2, 3])
def test_flux_equilibrium_and_mean_preservation(k):
    """acceptance.cpp:333-392: solve paper-sine on a 4^3 box on the GPU, then
    the numerical flux of the recovered solution is single-valued on every
    interior face (its moments against the complete P_k face basis cancel
    between the two sides, residual / scale < 1e-8) and the postprocess keeps
    the element means (|u*_0 - u_0| < 1e-12)."""
    prob = PAPER_SINE
    mesh = HostMesh.box(4, bc=prob.bc)
    em = oracle_mesh(mesh)
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    cs = eng.build_condense(g, prob.kappa, prob.c, prob.f)
    pat = eng.pattern_device(dm)
    sysH = eng.assemble(dm, pat, cs)
    eng.neumann_load(dm, g, prob.q, b=sysH.b, alpha=-1.0)
    ub = eng.dirichlet_project(dm, prob.u)
    uhat, _ = eng.solve_skeleton(dm, pat, sysH, ub, rtol=1e-14)
    ls = eng.recover(g, dm, cs, uhat)
    d2 = dim2(k)
    _, _, lb, _, _ = oracle_condense(em, k, prob.kappa, prob.c, prob.f, 1.0)
    uh = np_(uhat)
    lam = core.gather_traces(em, d2, uh)
    total = np.zeros((dm.nfc, d2))
    sides = np.zeros(dm.nfc, int)
    scale = 0.0
    fb = mesh.facebyele
    for K in range(em.n_elements):
        mom = _flux_moments(lb, ls, lam[:, K], K).reshape(4, d2)
        scale = max(scale, float(np.max(np.abs(mom))))
        for l in range(4):
            total[fb[K, l]] += mom[l]
            sides[fb[K, l]] += 1
    interior = sides == 2
    assert interior.sum() == dm.nfc - dm.ndir - dm.nneu
    assert np.max(np.abs(total[interior])) / scale < 1e-8
    eng.set_postprocess_rule()
    ustar = eng.postprocess_star(g, prob.kappa, ls)
    assert float((ustar[:, 0] - ls.u[:, 0]).abs().max()) < 1e-12


def test_full_size_properties_c2():
    """BASELINE C2 at full size (196,608 tets, k = 3): properties that need no
    oracle re-solve. (1) every C is symmetric to rounding; (2) the recovery is
    affine in lambda: R(a + b) - R(a) - R(b) + R(0) = 0; (3) the postprocess
    preserves the element means; (4) checksum of checksums: the sum of all
    entries of the assembled H and b equals the sum over the elements' C and
    Cf (Dirichlet rows included: assemble adds every contribution,
    global_system.cpp:31-56)."""
    cfg = CONFIGS["C2"]
    prob = cfg.problem
    mesh = HostMesh.box(cfg.n, bc=prob.bc, perturb=cfg.perturb, seed=cfg.seed)
    k = cfg.k
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, cfg.tau)
    cs = eng.build_condense(g, prob.kappa, prob.c, prob.f)
    C = cs.C_slices()
    nrm = C.abs().amax(dim=(1, 2))
    asym = (C - C.transpose(1, 2)).abs().amax(dim=(1, 2)) / nrm
    assert float(asym.max()) < 1e-12
    d2 = dim2(k)
    gen = torch.Generator(device="cuda").manual_seed(3)
    a = torch.rand(dm.nfc * d2, dtype=torch.float64, device="cuda", generator=gen) - 0.5
    b = torch.rand(dm.nfc * d2, dtype=torch.float64, device="cuda", generator=gen) - 0.5
    def rec(x):
        ls = eng.recover(g, dm, cs, x)
        return torch.stack([ls.qx.clone(), ls.qy.clone(), ls.qz.clone(), ls.u.clone()])
    r0, ra, rb, rab = rec(torch.zeros_like(a)), rec(a), rec(b), rec(a + b)
    scale = float(rab.abs().max())
    assert float((rab - ra - rb + r0).abs().max()) < 1e-11 * scale
    ls = eng.recover(g, dm, cs, a)
    eng.set_postprocess_rule()
    ustar = eng.postprocess_star(g, prob.kappa, ls)
    assert float((ustar[:, 0] - ls.u[:, 0]).abs().max()) < 1e-12 * max(1.0, float(ls.u[:, 0].abs().max()))
    pat = eng.pattern_device(dm)
    sysH = eng.assemble(dm, pat, cs)
    sum_abs = float(C.abs().sum())
    assert abs(float(sysH.vals.sum()) - float(C.sum())) < 1e-12 * sum_abs
    Cf = cs.Cf_cols()
    assert abs(float(sysH.b.sum()) - float(Cf.sum())) < 1e-12 * float(Cf.abs().sum())


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_chat_sparsity_kernels_agree(k):
    """K3 with the structurally zero blocks of Chat_# skipped (default) against
    the dense instantiation of the same kernel (hdg_b200_set_chat_sparsity 0)
    and against the oracle, on a perturbed mesh with every perm code in play:
    both within the parity tolerance, and within rounding of each other."""
    n = 2 if k < 4 else 1
    mesh = HostMesh.box(n, bc="dirichlet_x", perturb=0.1, seed=9)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    assert eng.set_chat_sparsity(True) is True  # the tables have the pattern
    d2 = dim2(k)
    rng = np.random.default_rng(3)
    uhat = torch.from_numpy(rng.standard_normal(dm.nfc * d2)).cuda()
    ls = eng.recover(g, dm, cs, uhat)
    sparse = [cs.C.clone(), cs.Cf.clone(), ls.u.clone(), ls.qx.clone()]
    assert eng.set_chat_sparsity(False) is False
    cs2 = eng.build_condense(g, KAP, CC, FF)
    ls2 = eng.recover(g, dm, cs2, uhat)
    dense = [cs2.C, cs2.Cf, ls2.u, ls2.qx]
    for a, b in zip(sparse, dense):
        assert float((a - b).abs().max()) <= 1e-12 * float(b.abs().max())
    _, _, lb, C, Cf = oracle_condense(em, k, KAP, CC, FF, 1.0)
    from oracle_util import max_slice_relerr
    for got in (cs, cs2):
        assert max_slice_relerr(np_(got.C_slices()), C) < 1e-10
        assert max_slice_relerr(np_(got.Cf_cols()), Cf.T) < 1e-10
