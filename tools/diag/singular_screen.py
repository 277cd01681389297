"""Evidence for the rescue screen of kernels_rescue.cuh (CPU, oracle + numpy).

For random elements (degrees 1..3, box meshes scaled to h = 1..1e-4, interior
jitter, kappa scaled by 1..1e20, c in [-1e4, 1e2], tau in [0, 100]/h) compare
the reference's singularity ratio min|U_ii| / max|U_ii| of A1's partial-pivot
LU (factor_checked, local_solver.cpp:50-57) with the screen's combined ratio
min / max over the |LDL^T pivots| of M and of S = D + sum_s C_s M^-1 C_s^T
(what the condensation kernels record). The screen is safe if the combined
ratio never exceeds the reference ratio by more than the screen's margin
(1e-12 / 1e-14 = 100)."""
import os
import sys

import numpy as np
import scipy.linalg as sl

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from oracle import core  # noqa: E402
from oracle_util import field  # noqa: E402


def ldl_pivots(A):
    A = A.copy()
    p = []
    for i in range(A.shape[0]):
        p.append(A[i, i])
        if A[i, i] != 0:
            A[i + 1:, i + 1:] -= np.outer(A[i + 1:, i], A[i, i + 1:]) / A[i, i]
    return np.abs(np.array(p))


rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
worst = np.inf
rows = []
for trial in range(int(sys.argv[2]) if len(sys.argv) > 2 else 60):
    k = int(rng.integers(1, 4))
    L = 10.0 ** -rng.uniform(0, 4)
    raw = core.box_mesh_raw(1, 1, 1, "all_dirichlet", [0, L, 0, L, 0, L])
    coords = np.array(raw[0])
    coords += rng.uniform(-0.1, 0.1, coords.shape) * L   # jitter every vertex a little
    raw = (np.asfortranarray(coords),) + tuple(raw[1:])
    try:
        em = core.expand(*raw)
    except Exception:
        continue
    kap = f"{10.0 ** rng.uniform(0, 20)!r} * (1 + 0.5*sin(x/{L!r}))"
    c = f"{rng.uniform(-1e4, 1e2)!r}"
    tau = rng.uniform(0, 100) / L
    t = core.tables(k, 2 * k + 2, 2 * k + 2)
    ms = core.build_element_matrices(em, t, field(kap), field(c), field("1"),
                                     core.Stabilization(np.full((em.n_elements, 4), tau)))
    lb = core.local_blocks(ms)
    d3 = (k + 1) * (k + 2) * (k + 3) // 6
    for K in range(em.n_elements):
        A1 = lb.A1[K]
        lu, _ = sl.lu_factor(A1, check_finite=False)
        d = np.abs(np.diag(lu))
        ref = d.min() / d.max()
        M = A1[:d3, :d3]
        Cb = A1[3 * d3:, :3 * d3]
        D = A1[3 * d3:, 3 * d3:]
        Mi = np.linalg.inv(M)
        S = D + sum(Cb[:, s * d3:(s + 1) * d3] @ Mi @ Cb[:, s * d3:(s + 1) * d3].T for s in range(3))
        piv = np.r_[ldl_pivots(M), ldl_pivots(S)]
        comb = piv.min() / piv.max()
        rows.append((ref, comb))
        worst = min(worst, ref / comb)
rows = np.array(rows)
print(f"{len(rows)} elements: min(ref / combined) = {worst:.3e}; "
      f"ref < 1e-14 in {int((rows[:, 0] < 1e-14).sum())}, combined < 1e-12 in {int((rows[:, 1] < 1e-12).sum())}, "
      f"missed (ref < 1e-14 but combined >= 1e-12): {int(((rows[:, 0] < 1e-14) & (rows[:, 1] >= 1e-12)).sum())}")
