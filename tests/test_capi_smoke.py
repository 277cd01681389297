"""The compiled C++ client (tests/capi_smoke.cpp over include/hdg/b200.hpp and
include/hdg_b200.h): its outputs match the oracle, and it checks the
reference's exception contract itself (exit code)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import core
from oracle_util import field, max_slice_relerr
from paper_1305_1489_b200.engine import HostMesh

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "capi_smoke")


def test_capi_smoke_binary_built_and_linked():
    assert os.path.exists(BIN), "tests/capi_smoke not built (__graft_entry__.build)"
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libhdg_b200.so" in out and "not found" not in out.split("libhdg_b200.so")[1].splitlines()[0]


@pytest.mark.gpu
def test_capi_smoke_matches_oracle(tmp_path):
    out = tmp_path / "capi.bin"
    r = subprocess.run([BIN, str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    raw = np.fromfile(out, dtype=np.uint8)
    nelt, m, d3, d3p = np.frombuffer(raw[:16].tobytes(), dtype=np.int32)
    v = np.frombuffer(raw[16:].tobytes(), dtype=np.float64)
    sizes = [nelt * m * m, nelt * m] + [nelt * d3] * 4 + [nelt * d3p]
    parts = np.split(v, np.cumsum(sizes)[:-1])
    C = parts[0].reshape(nelt, m, m).transpose(0, 2, 1)       # slice K column-major
    Cf, qx, qy, qz, u, us = (p.reshape(-1, r).T for p, r in zip(parts[1:], [m, d3, d3, d3, d3, d3p]))
    k = 2
    mesh = HostMesh.box(2, bc="dirichlet_top_bottom")
    em = core.expand(mesh.coordinates, mesh.elements, mesh.dirichlet, mesh.neumann)
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    kap = field("2 + sin(x)*sin(y)*sin(z)")
    ms = core.build_element_matrices(em, t, kap, field("1 + 0.5*(x*x + y*y + z*z)"), field("cos(x + 2*y - z)"),
                                     core.Stabilization(np.ones((em.n_elements, 4))))
    lb = core.local_blocks(ms)
    Co, Cfo = core.condense(lb)
    d2 = (k + 1) * (k + 2) // 2
    uhat = np.sin(0.37 * np.arange(em.n_faces * d2))
    qxo, qyo, qzo, uo = core.local_recover(lb, core.gather_traces(em, d2, uhat))
    t1 = core.tables(k + 1, 2 * (k + 1) + 2, 2 * k + 2)
    uso = core.postprocess_star(em, t1, kap, qxo, qyo, qzo, uo)
    assert max_slice_relerr(C, Co) < 1e-10
    for got, want in ((Cf, Cfo), (qx, qxo), (qy, qyo), (qz, qzo), (u, uo), (us, uso)):
        assert max_slice_relerr(got.T, want.T) < 1e-10
