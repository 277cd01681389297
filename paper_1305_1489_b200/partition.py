"""Element slabs for multi-GPU runs.

Elements of a Kuhn box are cell-major with z outermost (mesh.cpp:208-211), so
rank r of G owns the contiguous element range [r*E/G, (r+1)*E/G) — a z-slab.
A slab keeps the global face numbering order (local faces are the global faces
it touches, ascending), so its skeleton pattern maps back to the global one
bit-exactly; faces shared with a neighbouring slab are the interface faces.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .engine import DeviceMesh, HostMesh


@dataclass
class Slab:
    rank: int
    nranks: int
    elem_begin: int
    elem_end: int
    vert_global: np.ndarray   # local vertex -> global vertex
    face_global: np.ndarray   # local face -> global face (ascending)
    interface: np.ndarray     # local ids of faces shared with another slab
    interface_rank: np.ndarray  # rank owning the other side of each interface face
    coords: np.ndarray        # (nver_local, 3)
    elements: np.ndarray      # (nelt_local, 4) local vertex ids
    faces: np.ndarray         # (nfc_local, 3) local vertex ids, global parametrisation
    facebyele: np.ndarray     # (nelt_local, 4) local face ids
    facetype: np.ndarray


def slab(mesh: HostMesh, rank: int, nranks: int) -> Slab:
    nelt = mesh.n_elements
    if nelt % nranks:
        raise ValueError("element count must divide evenly into slabs")
    e0, e1 = rank * nelt // nranks, (rank + 1) * nelt // nranks
    el = mesh.elements[e0:e1]
    fbe = mesh.facebyele[e0:e1]
    vg, el_local = np.unique(el, return_inverse=True)
    fg, fbe_local = np.unique(fbe, return_inverse=True)
    vmap = np.full(mesh.dims["nver"], -1, np.int64)
    vmap[vg] = np.arange(len(vg))
    faces = vmap[mesh.faces[fg]]
    # a face is an interface face if an element outside the slab also touches it
    counts_in = np.bincount(fbe_local.reshape(-1), minlength=len(fg))
    ftype = mesh.facetype[fg]
    interface = np.flatnonzero((ftype == 0) & (counts_in == 1))
    # the rank on the other side: the face's element outside [e0, e1)
    all_f = mesh.facebyele.reshape(-1)
    all_e = np.repeat(np.arange(nelt), 4)
    order = np.argsort(all_f, kind="stable")
    fs, es = all_f[order], all_e[order]
    pos = np.searchsorted(fs, fg[interface])
    ea, eb = es[pos], es[np.minimum(pos + 1, len(es) - 1)]
    other = np.where((ea >= e0) & (ea < e1), eb, ea)
    irank = (other // (nelt // nranks)).astype(np.int32)
    return Slab(rank, nranks, e0, e1, vg, fg, interface, irank, mesh.coordinates[vg],
                el_local.reshape(el.shape).astype(np.int32), faces.astype(np.int32),
                fbe_local.reshape(fbe.shape).astype(np.int32), ftype)


def upload_slab(s: Slab, device: torch.device) -> DeviceMesh:
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).to(device, dt)
    return DeviceMesh(len(s.vert_global), s.elements.shape[0], len(s.face_global),
                      t(s.coords, torch.float64), t(s.elements, torch.int32), t(s.faces, torch.int32),
                      t(s.facebyele, torch.int32), torch.from_numpy(s.facetype).to(device))


def slab_pattern(s: Slab):
    """Skeleton sparsity of the slab's local faces (hdg_b200_pattern_build_raw)."""
    import ctypes as C
    from . import _lib as L
    nelt, nfc = s.facebyele.shape[0], len(s.face_global)
    fbe = np.asfortranarray(s.facebyele, dtype=np.int32)
    fb = np.zeros(nfc + 1, np.int64)
    nb = np.zeros((nfc, 8), np.int32)
    sl = np.zeros((nelt, 16), np.uint8)
    L.check(L.lib().hdg_b200_pattern_build_raw(nelt, nfc, fbe.ctypes.data, None, fb.ctypes.data,
                                               nb.ctypes.data, sl.ctypes.data))
    return fb, nb, sl
