"""Interface-face exchange between z-slabs.

Each rank scatters its slab into a slab-local CSR (local faces in global
order). Off-diagonal face blocks never straddle ranks (two tets share at most
one face), so the only shared data are the interface faces' d2 x d2 diagonal
blocks of H and their d2 entries of b: every rank sends its contributions to
the neighbour owning the other side and adds what it receives. Both sides end
with a + b == b + a, bit-identical to the single-GPU assembly (0 + a + b).
Transport is torch.distributed (NCCL over NVLink on GPUs, gloo on CPU).
"""
from __future__ import annotations

from typing import Dict, List

import numpy as np
import torch

from .partition import Slab


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
