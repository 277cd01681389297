"""Helpers for the GPU parity tests: run the CUDA path (through the C ABI) and
the CPU oracle on the same inputs."""
from __future__ import annotations

import numpy as np
import torch

from oracle import core
from oracle_util import field, max_slice_relerr, vfield
from paper_1305_1489_b200.engine import Engine, HostMesh, dim2, dim3

TOL = 1e-10  # max over elements of ||x_gpu - x_oracle||_F / ||x_oracle||_F


def np_(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def oracle_mesh(mesh: HostMesh):
    return core.expand(mesh.coordinates, mesh.elements, mesh.dirichlet, mesh.neumann)


def submesh(mesh: HostMesh, elems):
    """Disjoint-element sub-mesh for sampled parity at full size: the selected
    elements with every face listed as Dirichlet in its GLOBAL vertex order, so
    perm codes and face areas match the full mesh."""
    elems = np.asarray(elems)
    el = mesh.elements[elems]
    fb = mesh.facebyele[elems]
    faces = mesh.faces
    verts, inv = np.unique(el, return_inverse=True)
    coords = mesh.coordinates[verts]
    el_local = inv.reshape(el.shape).astype(np.int32)
    remap = {v: i for i, v in enumerate(verts)}
    d = np.array([[remap[v] for v in faces[f]] for f in fb.reshape(-1)], dtype=np.int32)
    return core.expand(np.asfortranarray(coords), np.asfortranarray(el_local), np.asfortranarray(d),
                       np.zeros((0, 3), np.int32))


def gpu_pipeline(mesh: HostMesh, k: int, kappa, c, f, tau=1.0, tet_deg=None, tri_deg=None, eng=None):
    eng = eng or Engine(0)
    eng.set_degree(k, tet_deg, tri_deg)
    dm = eng.upload(mesh)
    g = eng.geometry(dm, tau)
    cs = eng.build_condense(g, kappa, c, f)
    return eng, dm, g, cs


def oracle_condense(em, k, kappa, c, f, tau, tet_deg=None, tri_deg=None):
    t = core.tables(k, tet_deg or 2 * k + 2, tri_deg or 2 * k + 2)
    tauf = core.Stabilization(np.asfortranarray(tau) if isinstance(tau, np.ndarray)
                              else np.full((em.n_elements, 4), float(tau)))
    ms = core.build_element_matrices(em, t, field(kappa), field(c), field(f), tauf)
    lb = core.local_blocks(ms)
    C, Cf = core.condense(lb, 4)
    return t, ms, lb, C, Cf
