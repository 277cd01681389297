"""CPU checks of bench.py's reference arm (test infrastructure): the config
meshes come from the oracle alone and equal the product generator's bit for
bit; config C2's compiled callbacks equal its field programs; the chunked
whole-mesh CPU pipeline runs."""
import numpy as np
import pytest

from oracle import core
from oracle.meshes import config_mesh
from oracle_util import field
from paper_1305_1489_b200.configs import CONFIGS
from paper_1305_1489_b200.engine import HostMesh


@pytest.mark.parametrize("n,bc,perturb", [(4, "dirichlet_x", 0.0), (6, "dirichlet_top_bottom", 0.15),
                                          (24, "dirichlet_top_bottom", 0.15)])
def test_config_mesh_matches_product_generator(n, bc, perturb):
    coords, elements, dirichlet, neumann = config_mesh(n, bc, perturb, 1305)
    hm = HostMesh.box(n, bc=bc, perturb=perturb, seed=1305)
    assert np.array_equal(coords, hm.coordinates)
    assert np.array_equal(elements, hm.elements)
    assert np.array_equal(dirichlet, hm.dirichlet) and np.array_equal(neumann, hm.neumann)


def test_c2_native_fields_match_programs():
    prob = CONFIGS["C2"].problem
    native = core.c2_native_fields()
    progs = [field(prob.kappa), field(prob.c), field(prob.f)]
    rng = np.random.default_rng(5)
    for x, y, z in rng.random((200, 3)):
        for a, b in zip(native, progs):
            va, vb = a(x, y, z), b(x, y, z)
            assert abs(va - vb) <= 1e-14 * max(1.0, abs(vb))


def test_chunked_pipeline_runs():
    em = core.expand(*config_mesh(3, "dirichlet_x"))
    k = 2
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    d2 = (k + 1) * (k + 2) // 2
    tau = core.Stabilization(np.ones((em.n_elements, 4)))
    uhat = np.asfortranarray(np.sin(np.arange(4 * d2 * em.n_elements, dtype=float)).reshape(4 * d2, -1, order="F"))
    kap, c, f = core.c2_native_fields()
    secs, chk = core.time_pipeline_chunked(em, t, kap, c, f, tau, uhat, 4, 16)
    assert secs > 0 and np.isfinite(chk)
