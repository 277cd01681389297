"""GPU parity on ragged element counts: meshes made of the first n tets of a
perturbed Kuhn box (n = 1, 2, ... , not multiples of any kernel's elements per
CTA batch), so the last batch of the CTA-batched condensation / recovery
kernels is partial, and counts above 148 x batch so CTAs loop. Reference
edge case: a single-element mesh (tests/oracles.hpp reference_tet_mesh) and
the two-tet mesh of tests/test_global_system.cpp:13-23 are the smallest
inputs the reference's own tests run."""
import numpy as np
import pytest
import torch

from gpu_util import TOL, gpu_pipeline, np_, oracle_condense, oracle_mesh
from oracle import core
from oracle_util import field, max_slice_relerr
from paper_1305_1489_b200.engine import HostMesh, dim2, dim3

pytestmark = pytest.mark.gpu

KAP = "2 + sin(x)*sin(y)*sin(z)"
CC = "1 + 0.5*(x*x + y*y + z*z)"
FF = "cos(x + 2*y - z)"
LOCAL_FACES = [(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)]


def first_tets(n: int, box: int) -> HostMesh:
    """The first n elements of a perturbed box, every boundary face Dirichlet."""
    full = HostMesh.box(box, bc="all_dirichlet", perturb=0.12, seed=7)
    el = full.elements[:n]
    keys = {}
    for e in range(n):
        for lf in LOCAL_FACES:
            tri = tuple(int(el[e, i]) for i in lf)
            keys.setdefault(tuple(sorted(tri)), []).append(tri)
    bnd = np.array([v[0] for v in keys.values() if len(v) == 1], dtype=np.int32)
    return HostMesh.from_raw(full.coordinates, el, bnd, np.zeros((0, 3), np.int32))


CASES = [(k, n) for k in range(6) for n in (1, 2, 7)] + \
        [(2, 1777), (3, 1483), (4, 151), (5, 149)]


@pytest.mark.parametrize("k,n", CASES)
def test_condense_and_recover_ragged(k, n):
    mesh = first_tets(n, 7 if n > 384 else 4)
    assert mesh.n_elements == n
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    t, ms, lb, C, Cf = oracle_condense(em, k, KAP, CC, FF, 1.0)
    assert max_slice_relerr(np_(cs.C_slices()), C) < TOL
    assert max_slice_relerr(np_(cs.Cf_cols()), Cf.T) < TOL
    # recovery from a random skeleton vector (gather_traces + local_recover)
    d2 = dim2(k)
    lam = np.random.default_rng(k * 1000 + n).standard_normal(dm.nfc * d2)
    ls = eng.recover(g, dm, cs, torch.from_numpy(lam).cuda())
    ref = core.local_recover(lb, core.gather_traces(em, d2, lam), 4)
    for got, want in zip((ls.qx, ls.qy, ls.qz, ls.u), ref):
        assert max_slice_relerr(np_(got), want.T) < TOL


@pytest.mark.parametrize("k,n", [(k, n) for k in range(5) for n in (1, 17)] + [(3, 1483)])
def test_postprocess_ragged(k, n):
    """postprocess_star (postprocess.cpp:33-74) on counts that leave a partial
    CTA batch (16 elements per CTA for k <= 3)."""
    from paper_1305_1489_b200.engine import LocalSolution
    mesh = first_tets(n, 7 if n > 384 else 4)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    eng.set_postprocess_rule()
    rng = np.random.default_rng(100 + k)
    arrs = [rng.standard_normal((n, dim3(k))) for _ in range(4)]
    us = eng.postprocess_star(g, KAP, LocalSolution(*(torch.from_numpy(a).cuda() for a in arrs)))
    t1 = core.tables(k + 1, 2 * (k + 1) + 2, 2 * k + 2)
    want = core.postprocess_star(em, t1, field(KAP), *(np.asfortranarray(a.T) for a in arrs))
    assert max_slice_relerr(np_(us), want.T) < TOL


@pytest.mark.parametrize("k", range(6))
def test_lowest_singular_element_across_ctas(k):
    """local_solver.cpp:89-98 (test_local_solver.cpp:279-290): the lowest
    singular element is reported, here with two singular elements far apart
    (different CTAs / batches of every condensation kernel)."""
    from paper_1305_1489_b200._lib import LocalSolverError
    from paper_1305_1489_b200.engine import Engine
    mesh = HostMesh.box(5)  # 750 tets
    eng = Engine(0)
    eng.set_degree(k)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, 1.0)
    X, _, _ = eng.quad_points(g)
    kap = torch.ones_like(X)
    kap[613] = float("inf")  # kappa^-1 = 0 -> M = 0 -> singular
    kap[401] = float("inf")
    with pytest.raises(LocalSolverError) as ei:
        eng.build_condense(g, kap.contiguous(), 1.0, 1.0)
    assert ei.value.element == 401
