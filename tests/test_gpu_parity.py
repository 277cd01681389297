"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs. Tolerance (BASELINE north star): numbering,
perm codes and the CSR pattern bit-exact; C, Cf, b, q, u, u* within 1e-10
relative (max over elements of the Frobenius relative error)."""
import numpy as np
import pytest
import torch

from gpu_util import TOL, gpu_pipeline, np_, oracle_condense, oracle_mesh, submesh
from oracle import core
from oracle_util import field, max_slice_relerr, relerr, solve_skeleton, vfield
from paper_1305_1489_b200.configs import CONFIGS, PAPER_SINE, scaled
from paper_1305_1489_b200.engine import Engine, HostMesh, dim2, dim3

pytestmark = pytest.mark.gpu

KAP = "2 + sin(x)*sin(y)*sin(z)"
CC = "1 + 0.5*(x*x + y*y + z*z)"
FF = "cos(x + 2*y - z)"


def perm_cover_host():
    coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1],
                       [2, 0, 0], [3, 0, 0], [2, 1, 0], [2, 0, 1]], dtype=float)
    elements = np.array([[0, 1, 2, 3], [4, 5, 6, 7]], dtype=np.int32)
    sigma = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    lf = [(0, 1, 2), (0, 1, 3), (0, 2, 3), (3, 1, 2)]
    d = np.zeros((8, 3), dtype=np.int32)
    for e in range(2):
        for l in range(4):
            s = sigma[(4 * e + l) % 6]
            d[4 * e + l] = [elements[e, lf[l][s[i]]] for i in range(3)]
    return HostMesh.from_raw(coords, elements, d, np.zeros((0, 3), np.int32))


# ----------------------------------------------------------------- K1
@pytest.mark.parametrize("which", ["box", "perturbed", "cover"])
def test_geometry(which):
    if which == "box":
        mesh = HostMesh.box(3, bc="dirichlet_x")
    elif which == "perturbed":
        mesh = HostMesh.box(4, bc="dirichlet_top_bottom", perturb=0.15, seed=1305)
    else:
        mesh = perm_cover_host()
    em = oracle_mesh(mesh)
    eng = Engine(0)
    eng.set_degree(1)
    dm = eng.upload(mesh)
    tau = torch.rand(4, dm.nelt, dtype=torch.float64, device="cuda") + 0.5
    g = eng.geometry(dm, tau)
    eng.synchronize()
    assert np.array_equal(np_(g.perm).T, em.perm)                       # bit-exact
    assert np.max(np.abs(np_(g.volume) - em.volume) / em.volume) < 1e-14
    assert np.max(np.abs(np_(g.area) - em.area) / em.area) < 1e-14
    assert np.max(np.abs(np_(g.normals).T - em.normals)) < 1e-15 * np.max(np.abs(em.normals)) * 10
    assert np.max(np.abs(np_(g.piola).T - core.piola_coefficients(em))) < 1e-14
    T = core.Stabilization(np.asfortranarray(np_(tau).T)).scaled(em)
    assert np.max(np.abs(np_(g.T).T - T)) < 1e-14


# ------------------------------------------------ a3-a5: element matrices
@pytest.mark.parametrize("k,which", [(1, "box"), (2, "cover"), (3, "box")])
def test_element_matrices(k, which):
    mesh = HostMesh.box(2) if which == "box" else perm_cover_host()
    em = oracle_mesh(mesh)
    eng, dm, g, _ = gpu_pipeline(mesh, k, KAP, CC, FF, tau=1.3)
    got = eng.element_matrices(g, KAP, CC, FF)
    _, ms, _, _, _ = oracle_condense(em, k, KAP, CC, FF, 1.3)
    for name in ("Mkinv", "Mc", "Cx", "Cy", "Cz", "tauPP", "tauDP", "nxDP", "nyDP", "nzDP", "tauDD"):
        want = ms.get(name)
        err = max_slice_relerr(np_(got[name]), want)
        assert err < TOL, (name, err)
    assert max_slice_relerr(np_(got["fvec"]), ms.get("fvec").T) < TOL


# ------------------------------------------------------ a8: condense
@pytest.mark.parametrize("k,n,bc", [(0, 2, "dirichlet_top_bottom"), (1, 3, "all_dirichlet"),
                                    (2, 2, "dirichlet_x"), (3, 2, "dirichlet_x"),
                                    (4, 1, "dirichlet_top_bottom"), (5, 1, "dirichlet_top_bottom")])
def test_condense(k, n, bc):
    mesh = HostMesh.box(n, bc=bc)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    _, _, _, C, Cf = oracle_condense(em, k, KAP, CC, FF, 1.0)
    assert max_slice_relerr(np_(cs.C_slices()), C) < TOL
    assert max_slice_relerr(np_(cs.Cf_cols()), Cf.T) < TOL


def test_condense_perm_cover_all_codes():
    mesh = perm_cover_host()
    em = oracle_mesh(mesh)
    assert set(np.unique(em.perm)) == {1, 2, 3, 4, 5, 6}
    eng, dm, g, cs = gpu_pipeline(mesh, 2, KAP, CC, FF)
    _, _, _, C, Cf = oracle_condense(em, 2, KAP, CC, FF, 1.0)
    assert max_slice_relerr(np_(cs.C_slices()), C) < TOL
    assert max_slice_relerr(np_(cs.Cf_cols()), Cf.T) < TOL


def test_condense_sampled_fields():
    """HDG_FIELD_SAMPLED: caller-evaluated callbacks at the device's nodes."""
    k = 2
    mesh = HostMesh.box(2)
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    X, Y, Z = eng.quad_points(g)
    kap = 2 + torch.sin(X) * torch.sin(Y) * torch.sin(Z)
    cc = 1 + 0.5 * (X * X + Y * Y + Z * Z)
    ff = torch.cos(X + 2 * Y - Z)
    cs = eng.build_condense(g, kap.contiguous(), cc.contiguous(), ff.contiguous())
    _, _, _, C, Cf = oracle_condense(oracle_mesh(mesh), k, KAP, CC, FF, 1.0)
    assert max_slice_relerr(np_(cs.C_slices()), C) < TOL
    assert max_slice_relerr(np_(cs.Cf_cols()), Cf.T) < TOL


def test_singular_element_reported():
    """local_solver.cpp:89-98 / test_local_solver.cpp:279-290: lowest singular index."""
    from paper_1305_1489_b200._lib import LocalSolverError
    k = 1
    mesh = HostMesh.box(2)
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    X, _, _ = eng.quad_points(g)
    kap = torch.ones_like(X)
    kap[3] = float("inf")   # kappa^-1 = 0 on element 3 -> M = 0 -> singular
    kap[7] = float("inf")
    with pytest.raises(LocalSolverError) as ei:
        eng.build_condense(g, kap.contiguous(), 1.0, 1.0)
    assert ei.value.element == 3


# ------------------------------------------------- a10: gather + recover
@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_recover(k):
    n = 2 if k < 5 else 1
    mesh = HostMesh.box(n, bc="dirichlet_x")
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    d2 = dim2(k)
    rng = np.random.default_rng(7)
    uhat = rng.standard_normal(dm.nfc * d2)
    ls = eng.recover(g, dm, cs, torch.from_numpy(uhat).cuda())
    _, _, lb, _, _ = oracle_condense(em, k, KAP, CC, FF, 1.0)
    qx, qy, qz, u = core.local_recover(lb, core.gather_traces(em, d2, uhat), 4)
    for got, want in ((ls.qx, qx), (ls.qy, qy), (ls.qz, qz), (ls.u, u)):
        assert max_slice_relerr(np_(got), want.T) < TOL


# ------------------------------------------------------ a9: scatter
@pytest.mark.parametrize("k,bc", [(1, "all_dirichlet"), (2, "dirichlet_x")])
def test_scatter_pattern_and_values(k, bc):
    mesh = HostMesh.box(3, bc=bc)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    pat = eng.pattern(mesh)
    sys = eng.assemble(dm, pat, cs)
    C = np_(cs.C_slices())
    Cf = np_(cs.Cf_cols()).T
    colptr, rowidx, vals, b = core.assemble(em, np.ascontiguousarray(C), np.asfortranarray(Cf))
    # pattern bit-exact (structurally symmetric: CSR(H) pattern == CSC(H) pattern)
    assert np.array_equal(np_(sys.rowptr), colptr)
    assert np.array_equal(np_(sys.colidx), rowidx)
    # values: CSR row r, col c == CSC entry (r, c) of H; compare via scipy
    import scipy.sparse as sp
    nd = len(b)
    Hg = sp.csr_matrix((np_(sys.vals), np_(sys.colidx), np_(sys.rowptr)), shape=(nd, nd))
    Ho = sp.csc_matrix((vals, rowidx, colptr), shape=(nd, nd))
    assert abs(Hg - Ho).max() <= 1e-13 * abs(Ho).max()
    assert np.max(np.abs(np_(sys.b) - b)) <= 1e-13 * np.max(np.abs(b))
    # two runs bit-identical, and the element-ordered K4 (fp64 atomics onto
    # zero on the diagonal blocks: a + b commutes) gives the same bits
    sys2 = eng.assemble(dm, pat, cs)
    assert torch.equal(sys.vals, sys2.vals) and torch.equal(sys.b, sys2.b)
    sys3 = eng.assemble(dm, pat, cs, by="elements")
    assert torch.equal(sys.vals, sys3.vals) and torch.equal(sys.b, sys3.b)


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4, 5])
def test_scatter_by_faces_matches_by_elements(k):
    """Face-ordered K4 == element-ordered K4 bit for bit, every degree, with a
    mixed-BC mesh (one- and two-sided faces) and random C, Cf."""
    mesh = HostMesh.box(2, 2, 3, bc="dirichlet_x")
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    pat = eng.pattern_device(dm)
    d2 = (k + 1) * (k + 2) // 2
    m = 4 * d2
    gen = torch.Generator(device="cuda").manual_seed(7 + k)
    Cr = torch.randn(dm.nelt, m, m, dtype=torch.float64, device="cuda", generator=gen)
    Cr = (Cr + Cr.transpose(1, 2)).contiguous()  # K4 by faces relies on C's symmetry (as the reference's H does)
    Cf = torch.randn(dm.nelt, m, dtype=torch.float64, device="cuda", generator=gen)
    from paper_1305_1489_b200.engine import CondensedSystem
    cs = CondensedSystem(Cr.reshape(-1), Cf.reshape(-1), None, m)
    a = eng.assemble(dm, pat, cs, by="faces")
    b = eng.assemble(dm, pat, cs, by="elements")
    assert torch.equal(a.vals, b.vals) and torch.equal(a.b, b.b)


# ------------------------------------------------ a11: postprocess
@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_postprocess(k):
    mesh = HostMesh.box(2, 1, 3) if k % 2 else HostMesh.box(2)  # 36 tets: a partial 8-element batch
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    eng.set_postprocess_rule()
    rng = np.random.default_rng(11)
    d3 = dim3(k)
    arrs = [rng.standard_normal((em.n_elements, d3)) for _ in range(4)]
    from paper_1305_1489_b200.engine import LocalSolution
    ls = LocalSolution(*(torch.from_numpy(a).cuda() for a in arrs))
    us = eng.postprocess_star(g, KAP, ls)
    t1 = core.tables(k + 1, 2 * (k + 1) + 2, 2 * k + 2)
    want = core.postprocess_star(em, t1, field(KAP), *(np.asfortranarray(a.T) for a in arrs))
    assert max_slice_relerr(np_(us), want.T) < TOL


# ------------------------------------------------ a6: convection block
@pytest.mark.parametrize("k", [0, 1, 2, 3, 4, 5])
def test_convection_block(k):
    """convection_bilinear_matrices (convdiff.cpp:5-28): the CTA-batched DMMA
    kernel at k <= 3 (72 tets: a partial last batch of 16), warp per element beyond."""
    mesh = HostMesh.box(2, 2, 3, perturb=0.1)
    em = oracle_mesh(mesh)
    beta = ("x*y", "y*z", "x + z*z")
    eng = Engine(0)
    eng.set_degree(k, 2 * k + 4, 2 * k + 4)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    vol, dp, dd = eng.convection_bilinear_matrices(g, beta)
    t = core.tables(k, 2 * k + 4, 2 * k + 4)
    v0, p0, d0 = core.convection_bilinear_matrices(em, t, vfield(beta))
    assert max_slice_relerr(np_(vol), v0) < TOL
    assert max_slice_relerr(np_(dp), p0) < TOL
    assert max_slice_relerr(np_(dd), d0) < TOL


# --------------------------------------------- K8: skeleton boundary data
@pytest.mark.parametrize("k", [0, 1, 3, 5])
def test_boundary_data(k):
    """dirichlet_project / neumann_load / l2_project_skeleton against the
    oracle on a perturbed box with Dirichlet and Neumann faces."""
    mesh = HostMesh.box(3, bc="dirichlet_x", perturb=0.1)
    em = oracle_mesh(mesh)
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    assert dm.ndir > 0 and dm.nneu > 0
    g = eng.geometry(dm, 1.0)
    qd, d2 = 2 * k + 2, dim2(k)
    u, q = "exp(x + y)*sin(3*z)", ("x*y - z", "cos(x*z)", "y + x*x")
    ub = np_(eng.dirichlet_project(dm, u))
    want = core.dirichlet_project(em, k, qd, field(u)).reshape(-1, d2)
    assert ub.shape == (dm.ndir, d2) and relerr(ub, want) < 1e-13
    nl = np_(eng.neumann_load(dm, g, q))
    want = core.neumann_load(em, k, qd, vfield(q))
    assert relerr(nl, want) < 1e-13
    assert not nl[:dm.ndir * d2].any() and not nl[(dm.ndir + dm.nneu) * d2:].any()
    b0 = torch.randn(dm.nfc * d2, dtype=torch.float64, device="cuda")
    b1 = np_(eng.neumann_load(dm, g, q, b=b0.clone(), alpha=-1.0))
    assert np.allclose(b1, np_(b0) - want, rtol=0, atol=1e-13)
    sk = np_(eng.skeleton_project(dm, u))
    want = core.l2_project_skeleton(em, k, qd, field(u)).T
    assert sk.shape == (dm.nfc, d2) and relerr(sk, want) < 1e-13


# ------------------------------------------------------ K9: skeleton solve
@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_solve_skeleton(k):
    """GPU block-Jacobi CG against the reference's direct solve of the same
    assembled system (global_system.cpp:106-165) on a perturbed mixed-BC mesh."""
    prob = CONFIGS["C2"].problem
    mesh = HostMesh.box(4, bc=prob.bc, perturb=0.1)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, prob.kappa, prob.c, prob.f)
    pat = eng.pattern_device(dm)
    sys = eng.assemble(dm, pat, cs)
    ub = eng.dirichlet_project(dm, prob.u)
    eng.neumann_load(dm, g, prob.q, b=sys.b, alpha=-1.0)
    uhat, info = eng.solve_skeleton(dm, pat, sys, ub)
    assert info["converged"] and info["relres"] <= 1e-13
    import scipy.sparse as sp
    nd = sys.b.numel()
    H = sp.csr_matrix((np_(sys.vals), np_(sys.colidx), np_(sys.rowptr)), shape=(nd, nd)).tocsc()
    want = solve_skeleton(em, H.indptr, H.indices, H.data, np_(sys.b), np_(ub).ravel(), dim2(k))
    assert relerr(np_(uhat), want) < 1e-10
    # Dirichlet dofs are the projected data, bit for bit
    assert np.array_equal(np_(uhat)[:ub.numel()], np_(ub).ravel())


@pytest.mark.parametrize("k", [0, 1, 2])
def test_solve_skeleton_nonsymmetric(k):
    """The reference's SparseLU branch (global_system.cpp:155-162): a system
    failing the symmetry test (here the assembled H with every value scaled by
    a smooth, non-symmetric factor, as an upwinded convection term would) is
    solved by the GPU BiCGStab and compared with the reference's direct solve."""
    prob = CONFIGS["C2"].problem
    mesh = HostMesh.box(3, bc=prob.bc, perturb=0.1)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, prob.kappa, prob.c, prob.f)
    pat = eng.pattern_device(dm)
    sys = eng.assemble(dm, pat, cs)
    idx = torch.arange(sys.vals.numel(), dtype=torch.float64, device="cuda")
    sys.vals.mul_(1.0 + 0.2 * torch.sin(0.7 * idx))
    ub = eng.dirichlet_project(dm, prob.u)
    uhat, info = eng.solve_skeleton(dm, pat, sys, ub, rtol=1e-12)
    assert info["converged"] and info["asym"] > 1e-3 * info["scale"]
    import scipy.sparse as sp
    nd = sys.b.numel()
    H = sp.csr_matrix((np_(sys.vals), np_(sys.colidx), np_(sys.rowptr)), shape=(nd, nd)).tocsc()
    want = solve_skeleton(em, H.indptr, H.indices, H.data, np_(sys.b), np_(ub).ravel(), dim2(k))
    assert relerr(np_(uhat), want) < 1e-9
    assert np.array_equal(np_(uhat)[:ub.numel()], np_(ub).ravel())


def test_solve_skeleton_singular_block_reported():
    """A vanished diagonal block of a nonsymmetric system: HDG_ESOLVE
    (GlobalSolverError, global_system.cpp:157-158)."""
    from paper_1305_1489_b200._lib import HdgError
    mesh = HostMesh.box(2, bc="dirichlet_x")
    eng, dm, g, cs = gpu_pipeline(mesh, 1, KAP, CC, FF)
    pat = eng.pattern_device(dm)
    sys = eng.assemble(dm, pat, cs)
    sys.vals[-2] += 1.0  # breaks H = H^T
    d2 = dim2(1)
    f = dm.nfc - 1  # last (interior) face: zero its whole block row
    fbase = pat.facebase.cpu().numpy()
    sys.vals[int(fbase[f]) * d2 * d2:int(fbase[f + 1]) * d2 * d2] = 0.0
    with pytest.raises(HdgError, match="factorization"):
        eng.solve_skeleton(dm, pat, sys, eng.dirichlet_project(dm, "x"))


# -------------------------------------------- end-to-end (C1 at full size)
def test_c1_full_pipeline_matches_oracle():
    """C1 (k=1, 8^3, 3072 tets): GPU condense -> scatter -> scipy solve ->
    GPU recover -> GPU postprocess reproduces the oracle's errors."""
    cfg = CONFIGS["C1"]
    prob = cfg.problem
    mesh = HostMesh.box(cfg.n, bc=prob.bc)
    em = oracle_mesh(mesh)
    k = cfg.k
    eng, dm, g, cs = gpu_pipeline(mesh, k, prob.kappa, prob.c, prob.f)
    pat = eng.pattern_device(dm)
    sys = eng.assemble(dm, pat, cs)
    # boundary data and the skeleton solve on the GPU (study.cpp:25-28)
    ub = eng.dirichlet_project(dm, prob.u)
    eng.neumann_load(dm, g, prob.q, b=sys.b, alpha=-1.0)
    uhat_d, info = eng.solve_skeleton(dm, pat, sys, ub)
    assert info["converged"] and info["asym"] < 1e-12 * info["scale"]
    uhat = np_(uhat_d)
    ls = eng.recover(g, dm, cs, uhat_d)
    eng.set_postprocess_rule()
    us = eng.postprocess_star(g, prob.kappa, ls)
    # oracle end to end
    from oracle_util import solve_level
    raw = (mesh.coordinates, mesh.elements, mesh.dirichlet, mesh.neumann)
    ref = solve_level(raw, k, prob)
    assert relerr(uhat, ref["uhat"]) < 1e-10
    assert max_slice_relerr(np_(ls.u), ref["u"].T) < 1e-9
    assert max_slice_relerr(np_(us), ref["ustar"].T) < 1e-9


# ---------------------------------------- full-size sampled parity (C2, C3)
@pytest.mark.parametrize("cfg_name", ["C2", "C3", "C4", "C5"])
def test_full_size_sampled_elements(cfg_name):
    """Full BASELINE mesh on the GPU; ~40 scattered elements re-solved by the
    oracle on a disjoint sub-mesh with the same face parametrisations (C4 with
    its upwind tau, C5 including the P_{k+1} postprocess)."""
    cfg = CONFIGS[cfg_name]
    prob = cfg.problem
    mesh = HostMesh.box(cfg.n, bc=prob.bc, perturb=cfg.perturb, seed=cfg.seed)
    k = cfg.k
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    tau = eng.upwind_tau(g, cfg.upwind_beta) if cfg.upwind_beta else cfg.tau
    g = eng.geometry(dm, tau)
    cs = eng.build_condense(g, prob.kappa, prob.c, prob.f)
    d2 = dim2(k)
    # lambda = face projection of u; here any smooth data works
    uhat = torch.sin(torch.arange(dm.nfc * d2, dtype=torch.float64, device="cuda") * 0.013)
    ls = eng.recover(g, dm, cs, uhat)
    nelt = dm.nelt
    sel = np.unique(np.linspace(0, nelt - 1, 40).astype(int))
    # keep elements pairwise non-adjacent
    fb = mesh.facebyele
    chosen, used = [], set()
    for K in sel:
        if used.isdisjoint(fb[K]):
            chosen.append(K)
            used.update(fb[K])
    sub = submesh(mesh, chosen)
    idx = torch.tensor(chosen, device="cuda")
    tau_sub = np_(tau)[:, chosen].T.copy() if isinstance(tau, torch.Tensor) else cfg.tau
    _, _, lb, C, Cf = oracle_condense(sub, k, prob.kappa, prob.c, prob.f, tau_sub)
    assert max_slice_relerr(np_(cs.C_slices()[idx]), C) < TOL
    assert max_slice_relerr(np_(cs.Cf_cols()[idx]), Cf.T) < TOL
    uh = np_(uhat)
    lam = np.stack([np.concatenate([uh[f * d2:(f + 1) * d2] for f in fb[K]]) for K in chosen], axis=1)
    qx, qy, qz, u = core.local_recover(lb, np.asfortranarray(lam), 4)
    assert max_slice_relerr(np_(ls.u[idx]), u.T) < TOL
    assert max_slice_relerr(np_(ls.qz[idx]), qz.T) < TOL
    if cfg.postprocess:
        eng.set_postprocess_rule()
        us = eng.postprocess_star(g, prob.kappa, ls)
        t1 = core.tables(k + 1, 2 * (k + 1) + 2, 2 * k + 2)
        want = core.postprocess_star(sub, t1, field(prob.kappa),
                                     *(np.asfortranarray(np_(x[idx]).T) for x in (ls.qx, ls.qy, ls.qz, ls.u)))
        assert max_slice_relerr(np_(us[idx]), want.T) < TOL


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_jit_and_interpreter_agree(k):
    """NVRTC-specialised node build == interpreted field programs (both GPU paths)
    at every block-size branch of the JIT kernel (256 threads below 100 nodes,
    384 at k = 3, 1024 at k >= 4); 107 tets leave a partial last CTA."""
    from test_gpu_ragged import first_tets
    mesh = first_tets(107, 3)
    prob = CONFIGS["C2"].problem
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    cs_jit = eng.build_condense(g, prob.kappa, prob.c, prob.f)
    assert eng.jit_status == "", eng.jit_status   # the compiled kernel ran (no silent fallback)
    eng.set_jit(False)
    cs_vm = eng.build_condense(g, prob.kappa, prob.c, prob.f)
    # fields differ only by FMA contraction in the compiled expressions (~1 ulp
    # of the node samples, amplified by cond(S) in Cf): the parity contract
    assert max_slice_relerr(np_(cs_jit.C_slices()), np_(cs_vm.C_slices())) < 1e-11
    assert max_slice_relerr(np_(cs_jit.Cf_cols()), np_(cs_vm.Cf_cols())) < 1e-10


@pytest.mark.parametrize("k", [2, 3])
def test_jit_samplers_run(k):
    """The NVRTC samplers of the postprocess kappa and the convection beta
    compile and run (a failure falls back silently to the interpreted
    programs: same values, several times slower), and the sampled paths agree
    with the interpreted ones."""
    from test_gpu_ragged import first_tets
    mesh = first_tets(107, 3)
    prob = CONFIGS["C2"].problem
    beta = CONFIGS["C4"].upwind_beta
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    cs = eng.build_condense(g, prob.kappa, prob.c, prob.f)
    uhat = torch.sin(torch.arange(dm.nfc * dim2(k), dtype=torch.float64, device="cuda") * 0.37)
    ls = eng.recover(g, dm, cs, uhat)
    eng.set_postprocess_rule()
    us = eng.postprocess_star(g, prob.kappa, ls)
    assert eng.jit_status == "", eng.jit_status
    conv = eng.convection_bilinear_matrices(g, beta)
    assert eng.jit_status == "", eng.jit_status
    eng.set_jit(False)
    us_vm = eng.postprocess_star(g, prob.kappa, ls)
    conv_vm = eng.convection_bilinear_matrices(g, beta)
    assert max_slice_relerr(np_(us), np_(us_vm)) < 1e-11
    for a, b in zip(conv, conv_vm):
        assert max_slice_relerr(np_(a), np_(b)) < 1e-12


# Field programs exercising the JIT emitter's rewrites (jit_quad.cpp
# FieldEmitter): sin/cos of exact multiples of pi as sinpi/cospi (m = 3, 1/2,
# -2, 2, 1), a non-multiple (pi*pi stays sin), folded literal products,
# subexpressions shared across kappa, c and f (sin(3*pi*x), sin(2*pi*x)), and
# the remaining operators (pow, sqrt, abs, lt, division, negation).
EMIT_FIELDS = [
    ("2 + sin(3*pi*x)*cos(pi/2*y)", "1 + 0.5*sin(pi*pi*z)**2",
     "cos(-2*pi*(x + y))*sin(3*pi*x) + sqrt(abs(x - y) + 1)"),
    ("1.5 + 0.25*lt(z, 0.5) + 0.5*sin(2*pi*x)", "exp(-x*y)",
     "(2 + sin(2*pi*x))/(1 + z*z) - cos(pi*z)**3"),
]


@pytest.mark.parametrize("kap,c,f", EMIT_FIELDS)
def test_jit_field_emitter_vs_oracle(kap, c, f):
    k = 2
    mesh = HostMesh.box(2, bc="dirichlet_x", perturb=0.1, seed=3)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, kap, c, f)
    assert eng.jit_status == "", eng.jit_status
    _, _, _, C, Cf = oracle_condense(em, k, kap, c, f, 1.0)
    assert max_slice_relerr(np_(cs.C_slices()), C) < TOL
    assert max_slice_relerr(np_(cs.Cf_cols()), Cf.T) < TOL


@pytest.mark.parametrize("nslabs,native", [(2, False), (2, True), (4, True)])
def test_two_slab_scatter_exchange_matches_global(nslabs, native):
    """z-slab scatter on the GPU (K4 into slab-local CSR) + interface exchange
    == the single-mesh GPU assembly, bit for bit. native: the
    C-ABI plan's gather / add kernels (hdg_b200_exchange_pack / _unpack_add,
    what hdg_b200_exchange_interface runs around its NCCL calls), the
    transport a device copy; 4 slabs give the middle ranks two neighbours."""
    from paper_1305_1489_b200.distributed import (NativeSlabExchange, SlabExchange, exchange_local,
                                                  exchange_local_native)
    from paper_1305_1489_b200.partition import slab, slab_pattern, upload_slab
    k = 2
    mesh = HostMesh.box(3, 3, 2 * nslabs, bc="dirichlet_x")
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    pat = eng.pattern(mesh)
    full = eng.assemble(dm, pat, cs)
    d2 = dim2(k)
    m = 4 * d2
    exs, systems, slabs = [], [], []
    for r in range(nslabs):
        s = slab(mesh, r, nslabs)
        fb, nb, sl = slab_pattern(s)
        sdm = upload_slab(s, torch.device("cuda"))
        sp_ = eng.pattern_from_arrays(fb, nb, sl)
        from paper_1305_1489_b200.engine import CondensedSystem
        n = s.elem_end - s.elem_begin
        scs = CondensedSystem(cs.C[s.elem_begin * m * m:s.elem_end * m * m], cs.Cf[s.elem_begin * m:s.elem_end * m],
                              None, m)
        ssys = eng.assemble(sdm, sp_, scs)
        exs.append(NativeSlabExchange(eng, s, fb, nb, d2) if native else SlabExchange(s, fb, nb, d2, torch.device("cuda")))
        systems.append((ssys.vals, ssys.b))
        slabs.append((s, fb, nb, ssys))
    (exchange_local_native if native else exchange_local)(exs, systems)
    import scipy.sparse as sp
    nd = dm.nfc * d2
    H = sp.csr_matrix((np_(full.vals), np_(full.colidx), np_(full.rowptr)), shape=(nd, nd))
    bg = np_(full.b)
    for s, fb, nb, ssys in slabs:
        fg = s.face_global
        vals, b = np_(ssys.vals), np_(ssys.b)
        rows = (fg[:, None] * d2 + np.arange(d2)).reshape(-1)
        assert np.array_equal(b, bg[rows])
        rp, ci = np_(ssys.rowptr), np_(ssys.colidx)
        gcols = (fg[ci // d2] * d2 + ci % d2)
        for lr in range(len(rows)):
            seg = slice(rp[lr], rp[lr + 1])
            want = np.asarray(H[rows[lr], gcols[seg]].todense()).ravel()
            assert np.array_equal(vals[seg], want)


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_condense_recover_perturbed(k):
    """The default condensation kernel (CTA-batched phases at k = 2, 3; one
    element per CTA iteration at k = 4, 5) and its recovery cache against the
    oracle's LU path on a perturbed mesh; 162 tets leave partial batches and
    > 148 CTAs' worth of iterations at k >= 4."""
    mesh = HostMesh.box(3, bc="dirichlet_x", perturb=0.1)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    d2 = dim2(k)
    uhat = torch.from_numpy(np.sin(np.arange(dm.nfc * d2) * 0.37)).cuda()
    ls = eng.recover(g, dm, cs, uhat)
    _, _, lb, C, Cf = oracle_condense(em, k, KAP, CC, FF, 1.0)
    assert max_slice_relerr(np_(cs.C_slices()), C) < TOL
    assert max_slice_relerr(np_(cs.Cf_cols()), Cf.T) < TOL
    qx, qy, qz, u = core.local_recover(lb, core.gather_traces(em, d2, uhat.cpu().numpy()), 4)
    for got, want in ((ls.qx, qx), (ls.qy, qy), (ls.qz, qz), (ls.u, u)):
        assert max_slice_relerr(np_(got), want.T) < TOL


@pytest.mark.parametrize("k", [1, 2, 3])
def test_recover_variants_agree(k):
    """TMA-streamed recovery (v3, default) and the direct-load kernel (v2) agree;
    1,296 tets spread over more warps than the persistent grid has, so every
    warp runs a chain of elements through both cache buffers."""
    mesh = HostMesh.box(6, bc="dirichlet_x", perturb=0.1)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    d2 = (k + 1) * (k + 2) // 2
    uhat = torch.from_numpy(np.sin(np.arange(dm.nfc * d2) * 0.37)).cuda()
    ls3 = eng.recover(g, dm, cs, uhat)
    eng.set_recover_variant(2)
    ls2 = eng.recover(g, dm, cs, uhat)
    for a, b in ((ls3.qx, ls2.qx), (ls3.qy, ls2.qy), (ls3.qz, ls2.qz), (ls3.u, ls2.u)):
        assert max_slice_relerr(np_(a), np_(b)) < 1e-12


# -------------------------------------------- a7: BDM variant (bdm_blocks)
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_bdm_variant(k):
    """bdm_blocks (local_solver.cpp:65-69): u truncated to P_{k-1}, tau ignored;
    C, Cf and the recovered (q, u) (u zero-padded) match the oracle."""
    mesh = HostMesh.box(2, bc="dirichlet_top_bottom", perturb=0.1)
    em = oracle_mesh(mesh)
    eng = Engine(0)
    eng.set_degree(k)
    eng.set_bdm(True)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)  # tau = 1 is ignored by the variant
    cs = eng.build_condense(g, KAP, CC, FF)
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    tauf = core.Stabilization(np.ones((em.n_elements, 4)))
    ms = core.build_element_matrices(em, t, field(KAP), field(CC), field(FF), tauf)
    lb = core.bdm_blocks(ms)
    C, Cf = core.condense(lb, 4)
    assert max_slice_relerr(np_(cs.C_slices()), C) < TOL
    assert max_slice_relerr(np_(cs.Cf_cols()), Cf.T) < TOL
    d2 = dim2(k)
    uhat = np.sin(np.arange(dm.nfc * d2) * 0.37)
    ls = eng.recover(g, dm, cs, torch.from_numpy(uhat).cuda())
    qx, qy, qz, u = core.local_recover(lb, core.gather_traces(em, d2, uhat), 4)
    for got, want in ((ls.qx, qx), (ls.qy, qy), (ls.qz, qz), (ls.u, u)):
        assert max_slice_relerr(np_(got), want.T) < TOL
    nu = dim3(k) - d2
    assert not np_(ls.u)[:, nu:].any()  # zero padding beyond P_{k-1}


def test_bdm_rejects_degree_zero():
    from paper_1305_1489_b200._lib import HdgError
    mesh = HostMesh.box(1)
    eng = Engine(0)
    eng.set_degree(0)
    eng.set_bdm(True)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 0.0)
    with pytest.raises(HdgError, match="k >= 1"):
        eng.build_condense(g, KAP, CC, FF)


def test_upwind_tau_independent():
    """Config C4's tau = 1 + |beta(x_e) . nu_{K,l}| against a host
    computation from the oracle's mesh: face centroid of local face l, unit
    outward normal from the oracle's area-scaled normals (mesh.cpp:153-169)."""
    cfg = CONFIGS["C4"]
    mesh = HostMesh.box(3, bc="all_dirichlet", perturb=0.12, seed=3)
    eng = Engine(0)
    eng.set_degree(2)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    tau = np_(eng.upwind_tau(g, cfg.upwind_beta))          # (4, nelt)
    em = oracle_mesh(mesh)
    X, el, nrm = em.coordinates, em.elements, em.normals
    lf = [(0, 1, 2), (0, 1, 3), (0, 2, 3), (3, 1, 2)]
    beta = lambda x, y, z: np.array([np.sin(np.pi * y), np.cos(np.pi * x), 0.5])
    assert cfg.upwind_beta == ("sin(pi*y)", "cos(pi*x)", "0.5")
    want = np.empty_like(tau)
    for K in range(em.n_elements):
        for l in range(4):
            xc = X[el[K, list(lf[l])]].sum(axis=0) / 3.0
            nu = nrm[K, 3 * l:3 * l + 3] / np.linalg.norm(nrm[K, 3 * l:3 * l + 3])
            want[l, K] = 1.0 + abs(beta(*xc) @ nu)
    assert np.max(np.abs(tau - want)) < 1e-13


def test_nccl_exchange_transport_self_peer():
    """hdg_b200_exchange_interface over real NCCL on one GPU: a one-rank
    communicator (unique id, comm init through the C ABI) and a plan whose
    neighbour is the rank itself, so the grouped ncclSend/ncclRecv returns each
    interface entry to its sender and the add doubles exactly those entries
    (every other CSR value and b entry untouched)."""
    import ctypes as C
    from paper_1305_1489_b200 import _lib as L
    from paper_1305_1489_b200.partition import slab, slab_pattern, upload_slab
    from paper_1305_1489_b200.engine import CondensedSystem
    from paper_1305_1489_b200.distributed import interface_positions
    k = 2
    mesh = HostMesh.box(3, 3, 4, bc="dirichlet_x")
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    d2 = dim2(k)
    m = 4 * d2
    s = slab(mesh, 0, 2)
    fb, nb, sl = slab_pattern(s)
    sdm = upload_slab(s, torch.device("cuda"))
    scs = CondensedSystem(cs.C[:s.elem_end * m * m], cs.Cf[:s.elem_end * m], None, m)
    sysH = eng.assemble(sdm, eng.pattern_from_arrays(fb, nb, sl), scs)
    v0, b0 = sysH.vals.clone(), sysH.b.clone()
    faces = np.ascontiguousarray(s.interface.astype(np.int32))
    fbc, nbc = np.ascontiguousarray(fb, np.int64), np.ascontiguousarray(nb, np.int32)
    plan = C.c_void_p()
    ranks, nf = np.array([0], np.int32), np.array([len(faces)], np.int32)
    L.check(L.lib().hdg_b200_exchange_plan(eng._ctx, len(fbc) - 1, d2, fbc.ctypes.data, nbc.ctypes.data, 1,
                                           ranks.ctypes.data, nf.ctypes.data, faces.ctypes.data, C.byref(plan)))
    uid = (C.c_ubyte * 128)()
    L.check(L.lib().hdg_b200_nccl_get_unique_id(uid))
    comm = C.c_void_p()
    L.check(L.lib().hdg_b200_nccl_comm_init(eng._ctx, 1, 0, uid, C.byref(comm)))
    try:
        L.check(L.lib().hdg_b200_exchange_interface(eng._ctx, plan, comm, sysH.vals.data_ptr(), sysH.b.data_ptr()))
        eng.synchronize()
    finally:
        L.lib().hdg_b200_nccl_comm_destroy(comm)
        L.lib().hdg_b200_exchange_free(plan)
    pos = interface_positions(fb, nb, faces, d2)
    nv = len(faces) * d2 * d2
    want_v, want_b = v0.clone(), b0.clone()
    want_v[torch.from_numpy(pos[:nv]).cuda()] *= 2
    want_b[torch.from_numpy(pos[nv:]).cuda()] *= 2
    assert torch.equal(sysH.vals, want_v) and torch.equal(sysH.b, want_b)
    assert len(faces) > 0
