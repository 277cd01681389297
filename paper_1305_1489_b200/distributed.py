"""Interface-face exchange between z-slabs.

Each rank scatters its slab into a slab-local CSR (local faces in global
order). Off-diagonal face blocks never straddle ranks (two tets share at most
one face), so the only shared data are the interface faces' d2 x d2 diagonal
blocks of H and their d2 entries of b: every rank sends its contributions to
the neighbour owning the other side and adds what it receives. Both sides end
with a + b == b + a, bit-identical to the single-GPU assembly (0 + a + b).
Two transports: `SlabExchange` (torch.distributed: NCCL over NVLink on GPUs,
gloo on CPU, the host-logic reference) and `NativeSlabExchange`, the engine's
own path through the C ABI (hdg_b200_exchange_plan / _interface: device
gather, one grouped ncclSend/ncclRecv per neighbour on the engine stream,
device add; include/hdg_b200.h).
"""
from __future__ import annotations

from typing import Dict, List

import numpy as np
import torch

from .partition import Slab


def interface_positions(facebase: np.ndarray, nbr: np.ndarray, faces: np.ndarray, d2: int) -> np.ndarray:
    """hdg_b200_exchange_positions: value positions of the faces' diagonal blocks,
    then their b positions (host only)."""
    import ctypes as C
    from . import _lib as L
    fb = np.ascontiguousarray(facebase, np.int64)
    nb = np.ascontiguousarray(nbr, np.int32)
    fc = np.ascontiguousarray(faces, np.int32)
    out = np.zeros(len(fc) * (d2 * d2 + d2), np.int64)
    L.check(L.lib().hdg_b200_exchange_positions(len(fb) - 1, d2, fb.ctypes.data, nb.ctypes.data, len(fc),
                                                fc.ctypes.data if len(fc) else None,
                                                out.ctypes.data if len(fc) else None))
    return out


def _diag_indices(facebase: np.ndarray, nbr: np.ndarray, faces: np.ndarray, d2: int):
    """CSR value positions of the diagonal blocks of `faces` and their b entries."""
    vals, bidx = [], []
    for f in faces:
        nb = int(facebase[f + 1] - facebase[f])
        s_self = int(np.flatnonzero(nbr[f, :nb] == f)[0])
        base = int(facebase[f]) * d2 * d2
        for i in range(d2):
            row = base + i * nb * d2 + s_self * d2
            vals.extend(range(row, row + d2))
            bidx.append(int(f) * d2 + i)
    return np.asarray(vals, np.int64), np.asarray(bidx, np.int64)


class SlabExchange:
    """Precomputed send/receive index sets of one slab, per neighbour rank."""

    def __init__(self, slab: Slab, facebase: np.ndarray, nbr: np.ndarray, d2: int, device):
        self.rank = slab.rank
        self.peers: Dict[int, tuple] = {}
        for q in np.unique(slab.interface_rank):
            faces = slab.interface[slab.interface_rank == q]   # ascending global order
            iv, ib = _diag_indices(facebase, nbr, faces, d2)
            self.peers[int(q)] = (torch.from_numpy(iv).to(device), torch.from_numpy(ib).to(device))

    def pack(self, q: int, vals: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        iv, ib = self.peers[q]
        return torch.cat([vals[iv], b[ib]])

    def unpack_add(self, q: int, buf: torch.Tensor, vals: torch.Tensor, b: torch.Tensor) -> None:
        iv, ib = self.peers[q]
        vals[iv] += buf[: iv.numel()]
        b[ib] += buf[iv.numel():]

    def exchange(self, vals: torch.Tensor, b: torch.Tensor, group=None) -> None:
        """Sum interface diagonal blocks and b with the neighbour slabs."""
        import torch.distributed as dist
        ops, recv = [], {}
        for q in sorted(self.peers):
            sbuf = self.pack(q, vals, b)
            rbuf = torch.empty_like(sbuf)
            recv[q] = rbuf
            ops.append(dist.P2POp(dist.isend, sbuf, q, group))
            ops.append(dist.P2POp(dist.irecv, rbuf, q, group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for q, rbuf in recv.items():
            self.unpack_add(q, rbuf, vals, b)


def exchange_local(exchanges: List[SlabExchange], systems: List[tuple]) -> None:
    """Single-process stand-in for `exchange` (all slabs in one process):
    systems[r] = (vals, b) of slab r."""
    bufs = {(r, q): ex.pack(q, *systems[r]) for r, ex in enumerate(exchanges) for q in ex.peers}
    for r, ex in enumerate(exchanges):
        for q in ex.peers:
            ex.unpack_add(q, bufs[(q, r)].to(systems[r][0].device), *systems[r])


class NativeSlabExchange:
    """The C-ABI exchange of one slab (hdg_b200_exchange_plan): per neighbour
    rank, the interface faces' diagonal-block and b positions in device memory."""

    def __init__(self, engine, slab: Slab, facebase: np.ndarray, nbr: np.ndarray, d2: int):
        import ctypes as C
        from . import _lib as L
        self.engine = engine
        self.peers = [int(q) for q in np.unique(slab.interface_rank)]
        faces = [slab.interface[slab.interface_rank == q].astype(np.int32) for q in self.peers]
        self.nfaces = [len(f) for f in faces]
        self.entries = [n * (d2 * d2 + d2) for n in self.nfaces]
        allf = np.ascontiguousarray(np.concatenate(faces) if faces else np.zeros(0, np.int32), np.int32)
        ranks = np.asarray(self.peers, np.int32)
        nf = np.asarray(self.nfaces, np.int32)
        fb = np.ascontiguousarray(facebase, np.int64)
        nb = np.ascontiguousarray(nbr, np.int32)
        h = C.c_void_p()
        L.check(L.lib().hdg_b200_exchange_plan(engine._ctx, len(fb) - 1, d2, fb.ctypes.data, nb.ctypes.data,
                                               len(self.peers), ranks.ctypes.data if len(ranks) else None,
                                               nf.ctypes.data if len(nf) else None,
                                               allf.ctypes.data if len(allf) else None, C.byref(h)))
        self._plan = h
        self._comm = None

    def __del__(self):
        from . import _lib as L
        if getattr(self, "_plan", None):
            L.lib().hdg_b200_exchange_free(self._plan)
            self._plan = None
        if getattr(self, "_comm", None):
            L.lib().hdg_b200_nccl_comm_destroy(self._comm)
            self._comm = None

    def init_comm(self, rank: int, world: int, group=None) -> None:
        """NCCL communicator of the engine's own: rank 0's unique id broadcast with
        torch.distributed (any backend)."""
        import ctypes as C
        import torch.distributed as dist
        from . import _lib as L
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            L.check(L.lib().hdg_b200_nccl_get_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        comm = C.c_void_p()
        L.check(L.lib().hdg_b200_nccl_comm_init(self.engine._ctx, world, rank, uid, C.byref(comm)))
        self._comm = comm

    def pack(self, i: int, vals: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        from . import _lib as L
        buf = torch.empty(self.entries[i], dtype=torch.float64, device=vals.device)
        L.check(L.lib().hdg_b200_exchange_pack(self.engine._ctx, self._plan, i, vals.data_ptr(), b.data_ptr(),
                                               buf.data_ptr()))
        return buf

    def unpack_add(self, i: int, buf: torch.Tensor, vals: torch.Tensor, b: torch.Tensor) -> None:
        from . import _lib as L
        L.check(L.lib().hdg_b200_exchange_unpack_add(self.engine._ctx, self._plan, i, buf.data_ptr(),
                                                     vals.data_ptr(), b.data_ptr()))

    def exchange(self, vals: torch.Tensor, b: torch.Tensor) -> None:
        """hdg_b200_exchange_interface on the engine stream (needs init_comm)."""
        from . import _lib as L
        L.check(L.lib().hdg_b200_exchange_interface(self.engine._ctx, self._plan, self._comm, vals.data_ptr(),
                                                    b.data_ptr()))


def exchange_local_native(exchanges: List[NativeSlabExchange], systems: List[tuple]) -> None:
    """Single-process stand-in for NativeSlabExchange.exchange (all slabs in one
    process, the transport a device copy): the C-ABI gather and add kernels."""
    bufs = {}
    for r, ex in enumerate(exchanges):
        for i, q in enumerate(ex.peers):
            bufs[(r, q)] = ex.pack(i, *systems[r])
    for r, ex in enumerate(exchanges):
        for i, q in enumerate(ex.peers):
            ex.unpack_add(i, bufs[(q, r)].to(systems[r][0].device), *systems[r])
