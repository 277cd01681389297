"""Pins the CPU oracle against the reference's own known-answer tests.

The reference library cannot be built here (no Eigen3), so the oracle is
pinned by porting the KATs of /root/reference/proj/tests (cited per test) and
the README golden error table (proj/README.md:78-82). These run on CPU.
"""
import math

import numpy as np
import pytest

from oracle import core
from oracle_util import box, field, relerr, solve_level, vfield
from paper_1305_1489_b200.configs import CONSTANT, PAPER_SINE, poly_k


def tet_monomial(a, b, c):  # tests/oracles.hpp:24-27
    return math.factorial(a) * math.factorial(b) * math.factorial(c) / math.factorial(a + b + c + 3)


def tri_monomial(a, b):  # tests/oracles.hpp:29-32
    return math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)


# ---------------------------------------------------------------- README golden
def test_readme_golden_errors():
    """proj/README.md:78-82: paper-sine, k=1, tau=1, levels 1-3 (n = 2, 4, 8)."""
    want_eq = [3.9548e-02, 1.0547e-02, 2.6813e-03]
    want_eu = [6.4292e-02, 1.6866e-02, 4.2920e-03]
    want_sizes = [(48, 120), (384, 864), (3072, 6528)]
    for lev, n in enumerate([2, 4, 8]):
        raw = core.box_mesh_raw(n, n, n, "dirichlet_top_bottom")
        r = solve_level(raw, 1, PAPER_SINE)
        assert (r["em"].n_elements, r["em"].n_faces) == want_sizes[lev]
        e = r["errors"]
        assert float(f"{e[0]:.4e}") == want_eq[lev]
        assert float(f"{e[1]:.4e}") == want_eu[lev]


# ------------------------------------------------------------------ quadrature
@pytest.mark.parametrize("deg", [0, 1, 2, 5, 8, 12])
def test_quadrature_exactness(deg):
    """tests/test_quadrature.cpp:49-67: exact to 1e-13 for monomials up to deg."""
    t = core.tables(0, deg, deg)
    bary, w = t.tet_bary, t.tet_w
    assert abs(w.sum() - 1.0) < 1e-14
    x, y, z = bary[:, 1], bary[:, 2], bary[:, 3]
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            for c in range(deg + 1 - a - b):
                got = (w * x**a * y**b * z**c).sum() / 6.0
                assert abs(got - tet_monomial(a, b, c)) < 1e-13
    tb, tw = t.tri_bary, t.tri_w
    s, tt = tb[:, 1], tb[:, 2]
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            assert abs((tw * s**a * tt**b).sum() / 2.0 - tri_monomial(a, b)) < 1e-13


@pytest.mark.parametrize("n,alpha", [(1, 0), (4, 1), (7, 2), (12, 0)])
def test_gauss_jacobi_against_numpy(n, alpha):
    """Golub-Welsch nodes vs numpy's Gauss-Legendre / scipy's Gauss-Jacobi."""
    from scipy.special import roots_jacobi
    x, w = core.gauss_jacobi01(n, alpha)
    xr, wr = roots_jacobi(n, alpha, 0.0)
    assert np.max(np.abs(x - (xr + 1) / 2)) < 2e-15
    assert np.max(np.abs(w - wr / 2.0 ** (alpha + 1))) < 2e-15


# ----------------------------------------------------------------------- basis
@pytest.mark.parametrize("k", [0, 1, 2, 3, 4, 5])
def test_basis_orthonormal(k):
    """tests/test_basis.cpp:33-49 + acceptance.cpp:253-267: Gram = 6I / 2I."""
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    G = t.P.T @ np.diag(t.tet_w) @ t.P
    assert np.max(np.abs(G - 6 * np.eye(t.d3))) < 1e-12
    Gd = t.D.T @ np.diag(t.tri_w) @ t.D
    assert np.max(np.abs(Gd - 2 * np.eye(t.d2))) < 1e-12
    assert abs(t.P[0, 0] - math.sqrt(6)) < 1e-14 and abs(t.D[0, 0] - math.sqrt(2)) < 1e-14


def test_basis_gradients_fd():
    """tests/test_basis.cpp: finite-difference gradients."""
    k = 3
    pts = np.array([[0.1, 0.2, 0.3], [0.25, 0.05, 0.6], [0.4, 0.3, 0.1]])
    Px, Py, Pz = core.eval_dubiner3d_grad(k, pts)
    h = 1e-6
    for d, G in enumerate((Px, Py, Pz)):
        e = np.zeros(3)
        e[d] = h
        fd = (core.eval_dubiner3d(k, pts + e) - core.eval_dubiner3d(k, pts - e)) / (2 * h)
        assert np.max(np.abs(fd - G)) < 1e-6


# ------------------------------------------------------------------------ mesh
def test_mesh_face_counts_and_perms():
    """tests/test_mesh.cpp: 48 elts, 120 faces; Kuhn perms are {1,3,5}."""
    _, em = box(2)
    assert em.n_elements == 48 and em.n_faces == 120
    assert set(np.unique(em.perm)) <= {1, 3, 5}
    assert np.all(em.volume > 0)
    # interior faces: normals of the two sides cancel
    fb, nrm = em.facebyele, em.normals
    acc = np.zeros((em.n_faces, 3))
    for K in range(em.n_elements):
        for l in range(4):
            acc[fb[K, l]] += nrm[K, 3 * l:3 * l + 3]
    interior = em.facetype == 0
    assert np.max(np.abs(acc[interior])) < 1e-15


def test_perm_cover_mesh_all_codes():
    """tests/oracles.hpp:241-259: two tets with boundary faces in all 6 orders."""
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
    em = core.expand(coords, elements, d, np.zeros((0, 3), dtype=np.int32))
    assert set(np.unique(em.perm)) == {1, 2, 3, 4, 5, 6}


def test_mesh_errors():
    """mesh.cpp:79-81: negative orientation rejected."""
    coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
    el = np.array([[0, 2, 1, 3]], dtype=np.int32)
    with pytest.raises(RuntimeError):
        core.expand(coords, el, np.zeros((0, 3), np.int32), np.zeros((0, 3), np.int32))


# ------------------------------------------------------------ element matrices
def test_mass_identity_and_source():
    """tests/test_element_matrices.cpp:49-53,82-89."""
    k = 2
    _, em = box(2)
    t = core.tables(k, 2 * k + 4, 2 * k + 2)
    M = core.mass_matrices(em, t, core.Field.constant(1.0))
    for K in range(em.n_elements):
        assert np.max(np.abs(M[K] - 6 * em.volume[K] * np.eye(t.d3))) < 1e-12
    ref = core.expand(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float),
                      np.array([[0, 1, 2, 3]], dtype=np.int32),
                      np.array([[0, 1, 2], [0, 1, 3], [0, 2, 3], [3, 1, 2]], dtype=np.int32),
                      np.zeros((0, 3), np.int32))
    f = core.source_vectors(ref, t, core.Field.constant(1.0))
    assert abs(f[0, 0] - math.sqrt(6) / 6) < 1e-13 and np.max(np.abs(f[1:, 0])) < 1e-13


def test_divergence_identity_and_surface_kats():
    """test_element_matrices.cpp:129-141 (C+C^T = type_a(n)), :220-228, :251-267, :287-299."""
    k = 2
    _, em = box(2)
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    Cs = core.convection_matrices(em, t)
    for s in range(3):
        B = core.type_a(em, t, core.normal_weights(em, s))
        assert np.max(np.abs(Cs[s] + np.transpose(Cs[s], (0, 2, 1)) - B)) < 1e-12
    area = em.area[em.facebyele]
    A = core.type_a(em, t, area)
    assert np.max(np.abs(A[:, 0, 0] - 6 * area.sum(1))) < 1e-12 * 6 * area.sum(1).max()
    Bb = core.type_b(em, t, area)
    d2 = t.d2
    for l in range(4):
        blk = Bb[:, l * d2:(l + 1) * d2, l * d2:(l + 1) * d2]
        assert np.max(np.abs(blk - 2 * area[:, l, None, None] * np.eye(d2))) < 1e-12
    Cc = core.type_c(em, t, area)
    for l in range(4):
        assert np.max(np.abs(Cc[:, l * d2, 0] - math.sqrt(12) * area[:, l])) < 1e-12


def test_stiffness_kernel():
    """test_element_matrices.cpp:356-367: constant mode is the 1-D kernel."""
    _, em = box(2)
    t = core.tables(2, 6, 6)
    S = core.stiffness_matrices(em, t)
    for K in range(0, em.n_elements, 7):
        assert np.max(np.abs(S[K][:, 0])) < 1e-12
        ev = np.linalg.eigvalsh(S[K])
        assert np.sum(np.abs(ev) < 1e-10) == 1 and ev.min() > -1e-10


# --------------------------------------------------------------- local solver
def _setup(k, kappa="1", c="1", f="1", tau=1.0, n=2):
    _, em = box(n)
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    tf = core.Stabilization(np.full((em.n_elements, 4), tau), allow_zero=(tau == 0.0))
    ms = core.build_element_matrices(em, t, field(kappa), field(c), field(f), tf)
    return em, t, ms


def test_flux_identity():
    """tests/test_local_solver.cpp:64-94 (<= 1e-10)."""
    k = 2
    em, t, ms = _setup(k, "2 + sin(x)*sin(y)*sin(z)", "1 + 0.5*(x*x + y*y + z*z)", "cos(x + 2*y - z)")
    lb = core.local_blocks(ms)
    C, Cf = core.condense(lb)
    rng = np.random.default_rng(7)
    uhat = np.asfortranarray(rng.standard_normal((4 * t.d2, em.n_elements)))
    qx, qy, qz, u = core.local_recover(lb, uhat)
    A3, DD = lb.A3, lb.tauDD
    for K in range(em.n_elements):
        qu = np.concatenate([qx[:, K], qy[:, K], qz[:, K], u[:, K]])
        lhs = -A3[K] @ qu + DD[K] @ uhat[:, K]
        rhs = C[K] @ uhat[:, K] - Cf[:, K]
        assert np.max(np.abs(lhs - rhs)) < 1e-10


def test_condensed_spd_and_threads():
    """test_local_solver.cpp:96-106 and :269-277 (bit-identical across threads)."""
    em, t, ms = _setup(1, "2", "1", "0")
    lb = core.local_blocks(ms)
    C1, Cf1 = core.condense(lb, 1)
    C4, Cf4 = core.condense(lb, 4)
    assert np.array_equal(C1, C4) and np.array_equal(Cf1, Cf4)
    for K in range(0, em.n_elements, 5):
        assert np.max(np.abs(C1[K] - C1[K].T)) < 1e-11
        assert np.linalg.eigvalsh(C1[K]).min() > -1e-11


def test_singular_element_reported():
    """test_local_solver.cpp:279-290."""
    em, t, ms = _setup(0)
    lb = core.local_blocks(ms)
    lb.zero_A1_slice(3)
    with pytest.raises(core.LocalSolverError) as ei:
        core.condense(lb)
    assert ei.value.args[1] == 3


def test_bdm_shapes():
    """test_local_solver.cpp:225-239."""
    em, t, ms = _setup(2, tau=0.0)
    lb = core.bdm_blocks(ms)
    assert lb.nu == t.d3 - t.d2 and lb.n == 3 * t.d3 + lb.nu
    assert np.max(np.abs(lb.tauDD)) == 0.0


# ---------------------------------------------------------------- pipeline
@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_poly_k_exactness(k):
    """tests/acceptance.cpp:115-133 / test_study.cpp:10-26: poly-k solved to 1e-9."""
    prob = poly_k(k, core.poly_k_terms(k))
    raw = core.box_mesh_raw(2, 2, 2, "dirichlet_top_bottom")
    r = solve_level(raw, k, prob)
    e = r["errors"]
    assert e[0] < 1e-9 and e[1] < 1e-9


def test_constant_problem():
    raw = core.box_mesh_raw(2, 2, 2, "dirichlet_top_bottom")
    r = solve_level(raw, 1, CONSTANT)
    assert r["errors"][1] < 1e-12


def test_postprocess_reproduces_kplus1():
    """tests/test_postprocess.cpp:40-63."""
    k = 1
    _, em = box(2)
    t1 = core.tables(k + 1, 2 * (k + 1) + 2, 2 * k + 2)
    hi = core.tables(k, 24, 24)
    kap = 2.0
    u = "1 + x*x - y*z + 2*z*z - x"
    qx = core.l2_project_volume(em, hi, field(f"-{kap}*(2*x - 1)"))
    qy = core.l2_project_volume(em, hi, field(f"{kap}*z"))
    qz = core.l2_project_volume(em, hi, field(f"-{kap}*(-y + 4*z)"))
    uu = core.l2_project_volume(em, hi, field(u))
    ustar = core.postprocess_star(em, t1, core.Field.constant(kap), qx, qy, qz, uu)
    hi1 = core.tables(k + 1, 24, 24)
    expect = core.l2_project_volume(em, hi1, field(u))
    assert np.max(np.abs(ustar - expect)) < 1e-10


def test_assembly_shared_face():
    """tests/test_global_system.cpp:46-82 (two-tet mesh)."""
    coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], dtype=float)
    el = np.array([[0, 1, 2, 3], [4, 3, 2, 1]], dtype=np.int32)
    d = np.array([[0, 1, 2], [0, 1, 3], [0, 2, 3], [4, 3, 2], [4, 3, 1], [4, 2, 1]], dtype=np.int32)
    em = core.expand(coords, el, d, np.zeros((0, 3), np.int32))
    t = core.tables(1, 4, 4)
    tf = core.Stabilization(np.ones((2, 4)))
    one = core.Field.constant(1.0)
    ms = core.build_element_matrices(em, t, one, one, one, tf)
    C, Cf = core.condense(core.local_blocks(ms))
    colptr, rowidx, vals, b = core.assemble(em, C, Cf)
    import scipy.sparse as sp
    nd = len(b)
    H = sp.csc_matrix((vals, rowidx, colptr), shape=(nd, nd)).toarray()
    assert np.max(np.abs(H - H.T)) < 1e-11
    fint = int(np.flatnonzero(em.facetype == 0)[0])
    l0 = list(em.facebyele[0]).index(fint)
    l1 = list(em.facebyele[1]).index(fint)
    d2 = 3
    s = C[0][l0 * d2:(l0 + 1) * d2, l0 * d2:(l0 + 1) * d2] + C[1][l1 * d2:(l1 + 1) * d2, l1 * d2:(l1 + 1) * d2]
    assert np.max(np.abs(H[fint * d2:(fint + 1) * d2, fint * d2:(fint + 1) * d2] - s)) < 1e-13
    sb = Cf[l0 * d2:(l0 + 1) * d2, 0] + Cf[l1 * d2:(l1 + 1) * d2, 1]
    assert np.max(np.abs(b[fint * d2:(fint + 1) * d2] - sb)) < 1e-13


def test_convdiff_constant_beta():
    """tests/test_convdiff.cpp:28-49."""
    k = 2
    _, em = box(2)
    t = core.tables(k, 2 * k + 4, 2 * k + 4)
    bx, by, bz = 1.5, -0.5, 2.0
    vol, dp, dd = core.convection_bilinear_matrices(
        em, t, core.VField(core.Field.constant(bx), core.Field.constant(by), core.Field.constant(bz)))
    Cx, Cy, Cz = core.convection_matrices(em, t)
    assert np.max(np.abs(vol - (bx * Cx + by * Cy + bz * Cz))) < 1e-12
    nw = [core.normal_weights(em, s) for s in range(3)]
    dpr = sum(b * core.type_c(em, t, n) for b, n in zip((bx, by, bz), nw))
    assert np.max(np.abs(dp - dpr)) < 1e-12
    ddr = core.type_b(em, t, bx * nw[0] + by * nw[1] + bz * nw[2])
    assert np.max(np.abs(dd - ddr)) < 1e-12
