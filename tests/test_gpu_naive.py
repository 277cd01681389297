"""The reference's acceptance criterion 6 (proj/tests/acceptance.cpp:137-239,
"batched kernels vs naive oracles") applied to the CUDA path: the materialised
ElementMatrixSet of the GPU (hdg_b200_element_matrices) against integrals
evaluated here in numpy on degree-20 rules through F_K^-1
(tests/oracles.hpp:96-103, 178-233), independently of the oracle's and the
product's table-driven assembly. The weights are polynomials of degree 2, so
the level's 2k+4 rules integrate every entry exactly and the two must agree
to rounding (the reference's bound: 1e-12)."""
import numpy as np
import pytest

from gpu_util import np_, oracle_mesh
from test_gpu_parity import perm_cover_host
from test_oracle_naive import face_points, naive_face_DP, phys_basis, phys_grad, tet_points
from paper_1305_1489_b200.engine import Engine, HostMesh

pytestmark = pytest.mark.gpu

MPT = "1 + 0.5*x - y + 2*z + 0.3*x*y"            # acceptance.cpp:143-145
KINV = "4 + 0.5*x - y + 2*z + 0.3*x*y"           # positive on both meshes: kappa = 1 / KINV


def _mpt(p, shift=0.0):
    return 1.0 + shift + 0.5 * p[:, 0] - p[:, 1] + 2.0 * p[:, 2] + 0.3 * p[:, 0] * p[:, 1]


def _relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("k,which", [(1, "box"), (2, "cover"), (3, "cover")])
def test_element_matrices_vs_naive_quadrature(k, which):
    mesh = HostMesh.box(2, bc="dirichlet_top_bottom") if which == "box" else perm_cover_host()
    em = oracle_mesh(mesh)   # mesh tables only (numbering, areas, normals): no oracle assembly below
    eng = Engine(0)
    eng.set_degree(k, 2 * k + 4, 2 * k + 4)
    dm = eng.upload(mesh)
    tau = 1.0 + 0.1 * (np.arange(em.n_elements)[None, :] + 2 * np.arange(4)[:, None])  # xi(K, l), acceptance.cpp:148-150
    import torch
    g = eng.geometry(dm, torch.from_numpy(np.ascontiguousarray(tau)).cuda())
    got = {n: np_(v) for n, v in eng.element_matrices(g, f"1/({KINV})", MPT, MPT).items()}
    d2 = (k + 1) * (k + 2) // 2
    worst = 0.0
    codes = set()
    for K in range(em.n_elements):
        pts, w, vol = tet_points(em, K)
        P = phys_basis(em, K, k, pts)
        dP = phys_grad(em, K, k, pts)
        wm, wk = vol * w * _mpt(pts), vol * w * _mpt(pts, 3.0)
        worst = max(worst, _relerr(got["Mc"][K], P.T @ (wm[:, None] * P)))
        worst = max(worst, _relerr(got["Mkinv"][K], P.T @ (wk[:, None] * P)))
        worst = max(worst, _relerr(got["fvec"][K], P.T @ wm))
        for s, name in enumerate(("Cx", "Cy", "Cz")):
            worst = max(worst, _relerr(got[name][K], P.T @ ((vol * w)[:, None] * dP[s])))
        # surface kernels against the per-face naive quadrature
        refT = np.zeros((4 * d2, P.shape[1]))
        refN = [np.zeros_like(refT) for _ in range(3)]
        refPP = np.zeros((P.shape[1], P.shape[1]))
        for l in range(4):
            f = em.facebyele[K, l]
            codes.add(int(em.perm[K, l]))
            ae = em.area[f]
            DP = naive_face_DP(em, K, l, k)
            refT[l * d2:(l + 1) * d2] = tau[l, K] * ae * DP
            for s in range(3):
                refN[s][l * d2:(l + 1) * d2] = em.normals[K, 3 * l + s] * DP
            phys, _, wf = face_points(em, f)
            Pf = phys_basis(em, K, k, phys)
            refPP += tau[l, K] * ae * (Pf.T @ (wf[:, None] * Pf))
        worst = max(worst, _relerr(got["tauDP"][K], refT))
        for s, name in enumerate(("nxDP", "nyDP", "nzDP")):
            worst = max(worst, _relerr(got[name][K], refN[s]))
        worst = max(worst, _relerr(got["tauPP"][K], refPP))
    assert worst < 1e-12, worst
    if which == "cover":
        assert codes == {1, 2, 3, 4, 5, 6}
