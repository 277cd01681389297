"""More of the reference's known-answer tests, ported to pin the oracle at
every degree the engine supports (k = 0..5; the reference's own KATs stop at
k = 1..3):

* trace pairing against the naive face oracle for every perm code
  (test_element_matrices.cpp:299-318, tests/oracles.hpp:162-233);
* the uncondensed single-element brute force (test_local_solver.cpp:142-223);
* polynomial exactness of the local solver (test_local_solver.cpp:108-140);
* poly-k exactness of the whole pipeline (acceptance.cpp:115-133) at k = 4, 5.

The naive integrals are evaluated here with numpy on degree-20 rules and the
physical basis through F_K^-1 (tests/oracles.hpp:96-103), independently of
the oracle's table-driven assembly.
"""
import numpy as np
import pytest

from oracle import core
from oracle_util import field, solve_level
from paper_1305_1489_b200.configs import poly_k

LF = [(0, 1, 2), (0, 1, 3), (0, 2, 3), (3, 1, 2)]   # mesh.hpp:38 kLocalFace


def perm_cover():
    """tests/oracles.hpp:241-259."""
    coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1],
                       [2, 0, 0], [3, 0, 0], [2, 1, 0], [2, 0, 1]], dtype=float)
    elements = np.array([[0, 1, 2, 3], [4, 5, 6, 7]], dtype=np.int32)
    sigma = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    d = np.zeros((8, 3), dtype=np.int32)
    for e in range(2):
        for l in range(4):
            s = sigma[(4 * e + l) % 6]
            d[4 * e + l] = [elements[e, LF[l][s[i]]] for i in range(3)]
    return core.expand(coords, elements, d, np.zeros((0, 3), dtype=np.int32))


def single_tet(coords):
    """reference_tet_mesh / skew_tet_mesh (tests/oracles.hpp:36-61)."""
    d = np.array([LF[l] for l in range(4)], dtype=np.int32)
    return core.expand(np.asarray(coords, float), np.array([[0, 1, 2, 3]], np.int32), d,
                       np.zeros((0, 3), np.int32))


SKEW = [[0.1, -0.2, 0.05], [1.3, 0.1, -0.3], [0.2, 1.1, 0.25], [-0.1, 0.3, 1.2]]


def _B(em, K):
    X = em.coordinates[em.elements[K]]
    return X[0], np.column_stack([X[1] - X[0], X[2] - X[0], X[3] - X[0]])


def phys_basis(em, K, k, pts):
    """tests/oracles.hpp:96-103: P_j at physical points through F_K^-1."""
    v1, B = _B(em, K)
    ref = (pts - v1) @ np.linalg.inv(B).T
    return core.eval_dubiner3d(k, np.asfortranarray(ref))


def phys_grad(em, K, k, pts):
    v1, B = _B(em, K)
    ref = (pts - v1) @ np.linalg.inv(B).T
    G = core.eval_dubiner3d_grad(k, np.asfortranarray(ref))
    Bit = np.linalg.inv(B).T
    return [sum(Bit[s, m] * G[m] for m in range(3)) for s in range(3)]


_TRI = core.tables(0, 2, 20)
_TET = core.tables(0, 20, 2)


def tet_points(em, K):
    v1, B = _B(em, K)
    ref = np.asarray(_TET.tet_bary)[:, 1:]
    return v1 + ref @ B.T, np.asarray(_TET.tet_w), abs(np.linalg.det(B)) / 6.0


def face_points(em, f):
    w = em.coordinates[em.faces[f]]
    st = np.asarray(_TRI.tri_bary)[:, 1:]
    return w[0] + st[:, :1] * (w[1] - w[0]) + st[:, 1:] * (w[2] - w[0]), st, np.asarray(_TRI.tri_w)


def naive_face_DP(em, K, l, k):
    """tests/oracles.hpp:185-211: (1/|e|) int_e D_i P_j over the face's own parametrisation."""
    f = em.facebyele[K, l]
    phys, st, w = face_points(em, f)
    D = core.eval_dubiner2d(k, np.asfortranarray(st))
    P = phys_basis(em, K, k, phys)
    return D.T @ (w[:, None] * P)


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4, 5])
def test_trace_pairing_matches_naive_face_every_perm(k):
    t = core.tables(k, 2 * k + 2, 2 * k + 4)
    d2 = t.d2
    seen = set()
    raw = core.box_mesh_raw(2, 2, 2, "dirichlet_top_bottom")
    for em in (core.expand(*raw), perm_cover()):
        xi = np.asfortranarray(em.area[em.facebyele])
        C = core.type_c(em, t, xi)
        for K in range(em.n_elements):
            for l in range(4):
                seen.add(int(em.perm[K, l]))
                ae = em.area[em.facebyele[K, l]]
                block = C[K][l * d2:(l + 1) * d2, :]
                assert np.max(np.abs(block - ae * naive_face_DP(em, K, l, k))) < 1e-11 * ae
    assert seen == {1, 2, 3, 4, 5, 6}


@pytest.mark.parametrize("k", [1, 3])
def test_uncondensed_single_element(k):
    """test_local_solver.cpp:142-223: A1 from naive integrals equals the
    batched assembly, and condense-free recovery solves the brute-force system."""
    kfun = lambda x, y, z: 1.0 + 0.3 * x + 0.2 * y * z
    em = single_tet(SKEW)
    t = core.tables(k, 2 * k + 6, 2 * k + 6)
    tau = core.Stabilization(np.full((1, 4), 2.0))
    ms = core.build_element_matrices(em, t, field("1 + 0.3*x + 0.2*y*z"), field("0.5"),
                                     field("1 + x - y + 2*z"), tau)
    lb = core.local_blocks(ms)
    d3, d2 = t.d3, t.d2
    # 1/kappa is not polynomial: the kernel's own rule (2k + 6), as the reference test does
    v1, B = _B(em, 0)
    tk = core.tables(0, 2 * k + 6, 2)
    pk = v1 + np.asarray(tk.tet_bary)[:, 1:] @ B.T
    wk = np.asarray(tk.tet_w) * abs(np.linalg.det(B)) / 6.0
    Pk = phys_basis(em, 0, k, pk)
    kinv = 1.0 / np.array([kfun(*p) for p in pk])
    Mk = Pk.T @ ((wk * kinv)[:, None] * Pk)
    pts, w, vol = tet_points(em, 0)
    P = phys_basis(em, 0, k, pts)
    wv = w * vol
    Mc = 0.5 * P.T @ (wv[:, None] * P)
    dP = phys_grad(em, 0, k, pts)
    Cs = [P.T @ (wv[:, None] * dP[s]) for s in range(3)]
    tpp = np.zeros((d3, d3))
    for l in range(4):
        f = em.facebyele[0, l]
        fp, _, fw = face_points(em, f)
        Pf = phys_basis(em, 0, k, fp)
        tpp += 2.0 * em.area[f] * Pf.T @ (fw[:, None] * Pf)
    A1 = np.zeros((4 * d3, 4 * d3))
    for s in range(3):
        A1[s * d3:(s + 1) * d3, s * d3:(s + 1) * d3] = Mk
        A1[s * d3:(s + 1) * d3, 3 * d3:] = -Cs[s].T
        A1[3 * d3:, s * d3:(s + 1) * d3] = Cs[s]
    A1[3 * d3:, 3 * d3:] = Mc + tpp
    assert np.max(np.abs(A1 - lb.A1[0])) < 1e-11
    gsk = core.l2_project_skeleton(em, k, 2 * k + 6, field("x*y - z"))
    uhat = np.asfortranarray(core.gather_traces(em, d2, np.ravel(gsk, order="F")))
    qx, qy, qz, u = core.local_recover(lb, uhat, 1)
    qu = np.concatenate([qx[:, 0], qy[:, 0], qz[:, 0], u[:, 0]])
    resid = A1 @ qu + lb.A2[0] @ uhat[:, 0] - lb.Af[:, 0]
    assert np.max(np.abs(resid)) < 1e-10


@pytest.mark.parametrize("k,u,grad,lap", [
    (2, "1 + x - 2*y + z + x*y - z*z", ("1 + y", "-2 + x", "1 - 2*z"), "-2"),
    (4, "1 + x - 2*y + z + x*y - z*z + x*x*y*y", ("1 + y + 2*x*y*y", "-2 + x + 2*x*x*y", "1 - 2*z"),
     "-2 + 2*y*y + 2*x*x"),
    (5, "1 + x*x*x*y*z - y*y*y*y*y + z*x", ("3*x*x*y*z + z", "x*x*x*z - 5*y*y*y*y", "x*x*x*y + x"),
     "6*x*y*z - 20*y*y*y"),
])
def test_local_polynomial_exactness(k, u, grad, lap):
    """test_local_solver.cpp:108-140 (k = 2 there; here also k = 4, 5): u in P_k,
    q = -kappa grad u, exact trace -> recovery returns the exact coefficients."""
    kap = 3.0
    raw = core.box_mesh_raw(2, 2, 2, "dirichlet_top_bottom")
    em = core.expand(*raw)
    qd = 2 * k + 2
    t = core.tables(k, qd, qd)
    f = f"-{kap!r}*({lap}) + ({u})"
    ms = core.build_element_matrices(em, t, field(str(kap)), field("1"), field(f),
                                     core.Stabilization(np.ones((em.n_elements, 4))))
    lb = core.local_blocks(ms)
    d2 = t.d2
    gsk = core.l2_project_skeleton(em, k, qd, field(u))
    uhat = np.asfortranarray(core.gather_traces(em, d2, np.ravel(gsk, order="F")))
    qx, qy, qz, uu = core.local_recover(lb, uhat, 1)
    th = core.tables(k, 2 * k + 4, qd)
    assert np.max(np.abs(uu - core.l2_project_volume(em, th, field(u)))) < 1e-10
    for got, g in zip((qx, qy, qz), grad):
        assert np.max(np.abs(got - core.l2_project_volume(em, th, field(f"-{kap!r}*({g})")))) < 1e-10


@pytest.mark.parametrize("k", [4, 5])
def test_poly_k_exactness_high_degree(k):
    """acceptance.cpp:115-133 at the degrees the engine adds (k = 4, 5)."""
    prob = poly_k(k, core.poly_k_terms(k))
    raw = core.box_mesh_raw(2, 2, 2, "dirichlet_top_bottom")
    e = solve_level(raw, k, prob)["errors"]
    assert e[0] < 1e-9 and e[1] < 1e-9
