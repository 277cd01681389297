"""CPU tests of the engine's host layer and C ABI (no GPU needed): the library
loads and exports every declared symbol; mesh numbering, perm-relevant face
triples, the skeleton pattern and the reference tables match the oracle."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import core
from paper_1305_1489_b200 import _lib as L
from paper_1305_1489_b200.configs import CONFIGS
from paper_1305_1489_b200.engine import HostMesh
from paper_1305_1489_b200.fields import compile_field

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hdg_b200.h")).read()
    declared = set(re.findall(r"\b(hdg_b200_\w+)\s*\(", hdr))
    lib = L.lib()
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(L.exported_symbols())
    assert lib.hdg_b200_version().decode().startswith("hdg_b200")


@pytest.mark.parametrize("n,bc", [(2, "dirichlet_top_bottom"), (3, "dirichlet_x"), (4, "all_dirichlet")])
def test_box_mesh_and_numbering_bit_exact(n, bc):
    raw = core.box_mesh_raw(n, n, n, bc)
    m = HostMesh.box(n, bc=bc)
    for a, b in zip(raw, (m.coordinates, m.elements, m.dirichlet, m.neumann)):
        assert np.array_equal(a, b)
    em = core.expand(*raw)
    assert np.array_equal(em.faces, m.faces)
    assert np.array_equal(em.facebyele, m.facebyele)
    assert np.array_equal(em.facetype, m.facetype)


def test_expand_perturbed_mesh_matches_oracle():
    cfg = CONFIGS["C3"]
    m = HostMesh.box(6, bc="dirichlet_top_bottom", perturb=cfg.perturb, seed=cfg.seed)
    co = m.coordinates
    assert np.any(co != core.box_mesh_raw(6, 6, 6, "dirichlet_top_bottom")[0])
    on_plane = np.isclose(core.box_mesh_raw(6, 6, 6, "dirichlet_top_bottom")[0][:, 2], 0.5)
    assert np.all(co[on_plane, 2] == 0.5)  # kappa jump stays element-aligned
    em = core.expand(co, m.elements, m.dirichlet, m.neumann)
    assert np.array_equal(em.faces, m.faces) and np.array_equal(em.facebyele, m.facebyele)
    assert np.all(em.volume > 0)


def test_expand_raw_mesh_and_errors():
    coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], dtype=float)
    el = np.array([[0, 1, 2, 3], [4, 3, 2, 1]], dtype=np.int32)
    d = np.array([[0, 1, 2], [0, 1, 3], [0, 2, 3], [4, 3, 2], [4, 3, 1], [4, 2, 1]], dtype=np.int32)
    m = HostMesh.from_raw(coords, el, d, np.zeros((0, 3), np.int32))
    em = core.expand(coords, el, d, np.zeros((0, 3), np.int32))
    assert np.array_equal(m.faces, em.faces) and np.array_equal(m.facebyele, em.facebyele)
    with pytest.raises(L.MeshError):  # missing boundary face (mesh.cpp:123-124)
        HostMesh.from_raw(coords, el, d[:5], np.zeros((0, 3), np.int32))
    with pytest.raises(L.MeshError):  # negative orientation (mesh.cpp:79-81)
        HostMesh.from_raw(coords, np.array([[0, 2, 1, 3]], np.int32), d[:3], np.zeros((0, 3), np.int32))


def test_pattern_matches_oracle_csc():
    k = 2
    d2 = 6
    m = HostMesh.box(3, bc="dirichlet_x")
    em = core.expand(m.coordinates, m.elements, m.dirichlet, m.neumann)
    fb, nb, sl = m.pattern()
    nelt = em.n_elements
    m4 = 4 * d2
    C = np.zeros((nelt, m4, m4))
    Cf = np.zeros((m4, nelt), order="F")
    colptr, rowidx, _, _ = core.assemble(em, C, Cf)
    # expand the compact pattern exactly as the device kernel does
    rowptr, colidx = [], []
    pos = 0
    for f in range(m.n_faces):
        n = fb[f + 1] - fb[f]
        for i in range(d2):
            rowptr.append(pos)
            for s in range(n):
                colidx.extend(nb[f, s] * d2 + np.arange(d2))
            pos += n * d2
    rowptr.append(pos)
    assert np.array_equal(np.array(rowptr), colptr)
    assert np.array_equal(np.array(colidx), rowidx)
    # slots point at the right neighbour
    fbe = m.facebyele
    for K in range(nelt):
        for l1 in range(4):
            for l2 in range(4):
                assert nb[fbe[K, l1], sl[K, 4 * l1 + l2]] == fbe[K, l2]


def _host_table(k, qd, which, n):
    out = np.zeros(n)
    L.check(L.lib().hdg_b200_host_table(k, qd, qd, L.TABLES[which], out.ctypes.data, n))
    return out


@pytest.mark.parametrize("k", [0, 1, 3, 5])
def test_tables_match_oracle(k):
    qd = 2 * k + 2
    t = core.tables(k, qd, qd)
    nq, d3, d2 = t.P.shape[0], t.d3, t.d2
    P = _host_table(k, qd, "P", nq * d3).reshape(nq, d3, order="F")
    assert np.max(np.abs(P - t.P)) < 1e-13
    w = _host_table(k, qd, "tet_w", nq)
    assert np.max(np.abs(w - t.tet_w)) < 1e-15
    bary = _host_table(k, qd, "tet_bary", nq * 4).reshape(nq, 4, order="F")
    assert np.max(np.abs(bary - t.tet_bary)) < 1e-15
    # Chat_# = (1/6)(wP)^T P_#  (element_matrices.cpp:117-122)
    Ch = _host_table(k, qd, "Chat", 3 * d3 * d3).reshape(3, d3, d3).transpose(0, 2, 1)
    for s, Pd in enumerate((t.Px, t.Py, t.Pz)):
        assert np.max(np.abs(Ch[s] - (np.diag(t.tet_w) @ t.P).T @ Pd / 6)) < 1e-13
    # W^{l,mu} = Dperm[mu]^T diag(w) Pface_l
    W = _host_table(k, qd, "Wlm", 24 * d2 * d3).reshape(24, d3, d2).transpose(0, 2, 1)
    for l in range(4):
        for mu in range(6):
            ref = t.Dperm(mu).T @ np.diag(t.tri_w) @ t.Pface(l)
            assert np.max(np.abs(W[6 * l + mu] - ref)) < 1e-13


def _c6_ch_nz(k, h, tile, s):
    """The condensation kernel's block mask (kernels_condense6.cuh, c6_ch_nz), restated."""
    if k == 3:
        if tile == 0:
            return not (h == 0 and s == 0)
        if tile == 1:
            return s == 4 or (h == 2 and s == 3)
        return False
    if k == 2:
        return tile == 0 and not (h == 0 and s == 0)
    return True


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_chat_structural_zeros(k):
    """The sparsity K3 relies on, on the reference's own tables (oracle) and on the
    product's host tables: Chat_h[i][j] = (1/6) int P_i d_h P_j (element_matrices.cpp:
    117-122) vanishes for i >= dim P_{k-1} and for j <= i; at k = 2, 3 every 8 x 4 operand
    block the kernel skips (c6_ch_nz, kidx kstep order) is zero, and every block it keeps
    is needed (the mask is tight)."""
    qd = 2 * k + 2
    t = core.tables(k, qd, qd)
    d3 = t.d3
    n1 = k * (k + 1) * (k + 2) // 6
    ref = [(np.diag(t.tet_w) @ t.P).T @ Pd / 6 for Pd in (t.Px, t.Py, t.Pz)]
    host = _host_table(k, qd, "Chat", 3 * d3 * d3).reshape(3, d3, d3).transpose(0, 2, 1)
    for Ch in (ref, host):
        mx = max(np.abs(c).max() for c in Ch)
        for c in Ch:
            assert np.abs(c[n1:, :]).max(initial=0.0) < 1e-13 * mx
            assert np.abs(np.tril(c)).max() < 1e-13 * mx
            # K3 v5 (k = 4, 5): a row tile's columns below its first row
            for tile in range((d3 + 7) // 8):
                assert np.abs(c[8 * tile:8 * tile + 8, :8 * tile]).max(initial=0.0) < 1e-13 * mx
        if k in (2, 3):
            npair = d3 // 8
            ks = 2 * npair + (1 if d3 % 8 else 0)
            for h, c in enumerate(Ch):
                for tile in range((d3 + 7) // 8):
                    for s in range(ks):
                        cols = [(s >> 1) * 8 + 2 * tt + (s & 1) if s < 2 * npair else 8 * npair + tt for tt in range(4)]
                        cols = [q for q in cols if q < d3]
                        blk = np.abs(c[8 * tile:min(8 * tile + 8, d3)][:, cols]).max(initial=0.0)
                        assert (blk > 1e-13 * mx) == _c6_ch_nz(k, h, tile, s), (h, tile, s, blk)


def test_field_compiler_roundtrip():
    for expr in ("1 + 0.5*sin(2*pi*x)*cos(2*pi*y)", "exp(x + y)*sin(pi*z)",
                 "(1 + 0.25*sin(2*pi*x)*sin(2*pi*y))*(100 - 99*lt(z, 0.5))", "x**2 - abs(y)/sqrt(2 + z)"):
        p = compile_field(expr)
        f = core.Field.program(p.ops, p.consts)
        for pt in ((0.1, 0.2, 0.3), (0.7, 0.4, 0.55), (0.9, 0.05, 0.45)):
            x, y, z = pt
            want = eval(expr.replace("lt(z, 0.5)", "(z < 0.5)"),
                        {"sin": np.sin, "cos": np.cos, "exp": np.exp, "pi": np.pi, "sqrt": np.sqrt,
                         "abs": abs, "x": x, "y": y, "z": z})
            assert abs(f(x, y, z) - want) < 1e-14 * max(1, abs(want))
            assert abs(float(p(x, y, z)) - want) < 1e-14 * max(1, abs(want))
    with pytest.raises(ValueError):
        compile_field("foo(x)")
