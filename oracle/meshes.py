"""TEST INFRASTRUCTURE ONLY: the BASELINE config meshes built from the oracle
alone (no product library), for bench.py's reference arm and the tests.

box_mesh is the oracle's restatement of the reference generator (mesh.cpp:
185-253). Config C3's interior jitter is builder-defined; this
is a plain-IEEE restatement of the product's generator
(paper_1305_1489_b200/csrc/host_mesh.cpp perturb_interior, compiled without
FMA contraction), bit-identical to it (tests/test_reference_arm.py).
"""
from __future__ import annotations

import numpy as np

from . import core

_MASK = (1 << 64) - 1


def _perturb(coords: np.ndarray, elements: np.ndarray, n: int, frac: float, seed: int,
             keep_plane_z: float = 0.5) -> np.ndarray:
    nv = n + 1
    h = 1.0 / n
    h3 = h * h * h
    X = np.array(coords, dtype=np.float64, order="C")
    inc = [[] for _ in range(len(X))]
    for K, vs in enumerate(elements):
        for v in vs:
            inc[v].append(K)
    state = [seed & _MASK]

    def uni() -> float:  # splitmix64 >> 11, scaled to [0, 1)
        s = (state[0] + 0x9E3779B97F4A7C15) & _MASK
        state[0] = s
        z = ((s ^ (s >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        z ^= z >> 31
        return float(z >> 11) * 2.0 ** -53

    def det(vv) -> float:
        B = [[X[vv[c + 1], r] - X[vv[0], r] for c in range(3)] for r in range(3)]
        return (B[0][0] * (B[1][1] * B[2][2] - B[2][1] * B[1][2]) -
                B[1][0] * (B[0][1] * B[2][2] - B[2][1] * B[0][2]) +
                B[2][0] * (B[0][1] * B[1][2] - B[1][1] * B[0][2]))

    for v in range(len(X)):
        i, j, k = v % nv, (v // nv) % nv, v // (nv * nv)
        if i in (0, n) or j in (0, n) or k in (0, n):
            continue
        x0, y0, z0 = (float(t) for t in X[v])
        on_plane = abs(z0 - keep_plane_z) < 1e-12
        for _ in range(16):
            dx = (2.0 * uni() - 1.0) * frac * h
            dy = (2.0 * uni() - 1.0) * frac * h
            dz = (2.0 * uni() - 1.0) * frac * h
            X[v] = (x0 + dx, y0 + dy, z0 if on_plane else z0 + dz)
            if all(det(elements[K]) > 0.25 * h3 for K in inc[v]):
                break
            X[v] = (x0, y0, z0)
    return X


def config_mesh(n: int, bc: str, perturb: float = 0.0, seed: int = 1305):
    """(coords, elements, dirichlet, neumann) of an n^3 Kuhn box, jittered like
    the product's HostMesh.box(n, bc=bc, perturb=perturb, seed=seed)."""
    coords, elements, dirichlet, neumann = core.box_mesh_raw(n, n, n, bc)
    if perturb > 0:
        coords = _perturb(coords, elements, n, perturb, seed)
    return (np.asfortranarray(coords), np.asfortranarray(elements), np.asfortranarray(dirichlet),
            np.asfortranarray(neumann))
