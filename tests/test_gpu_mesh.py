"""GPU mesh expansion and skeleton pattern against the host
restatement of mesh.cpp:74-171 / global_system.cpp:31-56: face numbering,
parametrisation, facetype, facebyele, facebase, neighbour lists and slots are
bit-exact; invalid meshes raise the same MeshError message."""
import numpy as np
import pytest
import torch

from gpu_util import np_
from paper_1305_1489_b200._lib import MeshError
from paper_1305_1489_b200.engine import Engine, HostMesh

pytestmark = pytest.mark.gpu


def raw_of(mesh):
    return mesh.coordinates, mesh.elements, mesh.dirichlet, mesh.neumann


def check_same(eng, mesh):
    dm = eng.expand(*raw_of(mesh))
    assert (dm.nfc, dm.ndir, dm.nneu) == (mesh.n_faces, mesh.dims["ndir"], mesh.dims["nneu"])
    assert np.array_equal(np_(dm.faces).T, mesh.faces)
    assert np.array_equal(np_(dm.facetype), mesh.facetype)
    assert np.array_equal(np_(dm.facebyele).T, mesh.facebyele)
    eng.set_degree(1)
    p = eng.pattern_device(dm)
    fb, nb, sl = mesh.pattern()
    assert np.array_equal(np_(p.facebase), fb)
    assert np.array_equal(np_(p.nbr), nb)
    assert np.array_equal(np_(p.slot), sl)
    q = eng.pattern(mesh)
    assert torch.equal(p.rowptr, q.rowptr) and torch.equal(p.colidx, q.colidx)
    return dm


@pytest.mark.parametrize("bc", ["all_dirichlet", "dirichlet_top_bottom", "dirichlet_x"])
@pytest.mark.parametrize("n,perturb", [(1, 0.0), (3, 0.0), (4, 0.12)])
def test_expand_matches_host(bc, n, perturb):
    check_same(Engine(0), HostMesh.box(n, bc=bc, perturb=perturb))


def test_expand_rectangular_and_full_size():
    eng = Engine(0)
    check_same(eng, HostMesh.box(2, 3, 5, bc="dirichlet_x"))
    check_same(eng, HostMesh.box(32, bc="dirichlet_x"))  # C2: 196,608 tets, 399,360 faces


def test_expand_perm_cover():
    from test_gpu_parity import perm_cover_host
    check_same(Engine(0), perm_cover_host())


def _host_error(*raw):
    with pytest.raises(MeshError) as e:
        HostMesh.from_raw(*raw)
    return str(e.value).split(":")[-1].strip()


def _device_error(eng, *raw):
    with pytest.raises(MeshError) as e:
        eng.expand(*raw)
    return str(e.value).split(":")[-1].strip()


def test_expand_errors_match_host():
    eng = Engine(0)
    mesh = HostMesh.box(2, bc="dirichlet_x")
    X, E, D, N = raw_of(mesh)
    cases = []
    e1 = E.copy()
    e1[5, [0, 1]] = e1[5, [1, 0]]  # inverted element
    cases.append((X, e1, D, N))
    cases.append((X, E, D[1:], N))  # boundary face not listed
    cases.append((X, E, np.vstack([D, D[:1]]), N))  # listed twice
    bogus = np.array([[0, 1, X.shape[0] - 1]], np.int32)
    cases.append((X, E, np.vstack([D, bogus]), N))  # matches no element face
    interior = mesh.faces[mesh.facetype == 0][:1]
    cases.append((X, E, np.vstack([D, interior]), N))  # shared by two elements
    for raw in cases:
        want = _host_error(*raw)
        got = _device_error(eng, *raw)
        assert got == want, (got, want)
