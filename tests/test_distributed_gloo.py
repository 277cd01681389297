"""Multi-rank host logic on CPU (gloo, world_size 2): z-slab partition,
slab-local skeleton patterns, and the interface-face exchange reproduce the
global assembly of the oracle. The per-element C, Cf come from
the oracle; the scatter here mirrors scatter_kernel's slot arithmetic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import core
from oracle_util import field
from paper_1305_1489_b200.engine import HostMesh
from paper_1305_1489_b200.partition import slab, slab_pattern

K_DEG, N = 1, 2


def _problem():
    mesh = HostMesh.box(N, N, 2 * N, bc="dirichlet_x")
    em = core.expand(mesh.coordinates, mesh.elements, mesh.dirichlet, mesh.neumann)
    t = core.tables(K_DEG, 2 * K_DEG + 2, 2 * K_DEG + 2)
    tau = core.Stabilization(np.ones((em.n_elements, 4)))
    ms = core.build_element_matrices(em, t, field("2 + x*y"), field("1 + z"), field("sin(x + y)"), tau)
    C, Cf = core.condense(core.local_blocks(ms))
    return mesh, em, C, Cf


def _scatter(s, fb, nb, sl, C, Cf, d2):
    """Host mirror of scatter_kernel into the slab-local CSR."""
    nfc = len(s.face_global)
    vals = np.zeros(int(fb[-1]) * d2 * d2)
    b = np.zeros(nfc * d2)
    m = 4 * d2
    for Kl in range(s.facebyele.shape[0]):
        K = s.elem_begin + Kl
        for l1 in range(4):
            f1 = s.facebyele[Kl, l1]
            n1 = fb[f1 + 1] - fb[f1]
            b[f1 * d2:(f1 + 1) * d2] += Cf[l1 * d2:(l1 + 1) * d2, K]
            for l2 in range(4):
                for i in range(d2):
                    pos = fb[f1] * d2 * d2 + i * n1 * d2 + sl[Kl, 4 * l1 + l2] * d2
                    vals[pos:pos + d2] += C[K][l1 * d2 + i, l2 * d2:(l2 + 1) * d2]
    return vals, b


def _check_against_global(s, fb, nb, vals, b, em, C, Cf, d2):
    colptr, rowidx, gvals, gb = core.assemble(em, np.ascontiguousarray(C), np.asfortranarray(Cf))
    import scipy.sparse as sp
    nd = len(gb)
    H = sp.csc_matrix((gvals, rowidx, colptr), shape=(nd, nd)).tocsr()
    fg = s.face_global
    for f in range(len(fg)):
        n1 = fb[f + 1] - fb[f]
        for i in range(d2):
            rg = fg[f] * d2 + i
            assert b[f * d2 + i] == gb[rg]   # bit-exact (a + b commutes)
            for sidx in range(n1):
                g = fg[nb[f, sidx]]
                for j in range(d2):
                    v = vals[fb[f] * d2 * d2 + i * n1 * d2 + sidx * d2 + j]
                    assert v == H[rg, g * d2 + j]


def _worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1305_1489_b200.distributed import SlabExchange
        mesh, em, C, Cf = _problem()
        d2 = (K_DEG + 1) * (K_DEG + 2) // 2
        s = slab(mesh, rank, world)
        fb, nb, sl = slab_pattern(s)
        vals, b = _scatter(s, fb, nb, sl, C, Cf, d2)
        tv, tb = torch.from_numpy(vals), torch.from_numpy(b)
        ex = SlabExchange(s, fb, nb, d2, torch.device("cpu"))
        assert set(ex.peers) == {1 - rank}
        ex.exchange(tv, tb)
        _check_against_global(s, fb, nb, tv.numpy(), tb.numpy(), em, C, Cf, d2)
        ret[rank] = 1
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_slab_partition_covers_mesh():
    mesh = HostMesh.box(N, N, 2 * N, bc="dirichlet_x")
    s0, s1 = slab(mesh, 0, 2), slab(mesh, 1, 2)
    assert s0.elem_end == s1.elem_begin == mesh.n_elements // 2
    shared = np.intersect1d(s0.face_global, s1.face_global)
    assert np.array_equal(shared, s0.face_global[s0.interface])
    assert np.array_equal(shared, s1.face_global[s1.interface])
    assert np.all(s0.interface_rank == 1) and np.all(s1.interface_rank == 0)
    assert len(shared) == 2 * N * N  # one z-plane of Kuhn cells: 2 triangles per cell


def test_two_rank_interface_exchange_gloo():
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), ret), nprocs=2, join=True)
    assert dict(ret) == {0: 1, 1: 1}


def test_native_interface_positions_match_host_logic():
    """hdg_b200_exchange_positions (the C-ABI plan's index sets) == the Python
    restatement used by the gloo exchange, for every slab of a 4-way split."""
    from paper_1305_1489_b200.distributed import _diag_indices, interface_positions
    mesh = HostMesh.box(N, N, 4 * N, bc="dirichlet_x")
    for k in (1, 3):
        d2 = (k + 1) * (k + 2) // 2
        for r in range(4):
            s = slab(mesh, r, 4)
            fb, nb, _ = slab_pattern(s)
            for q in np.unique(s.interface_rank):
                faces = s.interface[s.interface_rank == q]
                iv, ib = _diag_indices(fb, nb, faces, d2)
                assert np.array_equal(interface_positions(fb, nb, faces, d2), np.concatenate([iv, ib]))
