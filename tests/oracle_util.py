"""Test helpers around the CPU oracle (test infrastructure only)."""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import core
from paper_1305_1489_b200.configs import Problem
from paper_1305_1489_b200.fields import compile_field


def field(expr) -> "core.Field":
    try:
        p = compile_field(expr)
    except ValueError:  # beyond the device VM's limits (e.g. poly-k at k >= 4): a Python callback
        import math
        code = compile(str(expr), "<field>", "eval")
        env = {n: getattr(math, n) for n in ("sin", "cos", "exp", "sqrt", "pi")}
        return core.Field.python(lambda x, y, z: float(eval(code, env, {"x": x, "y": y, "z": z})))
    return core.Field.program(p.ops, p.consts)


def vfield(exprs) -> "core.VField":
    return core.VField(*(field(e) for e in exprs))


def box(n, bc="dirichlet_top_bottom", ny=None, nz=None):
    raw = core.box_mesh_raw(n, ny or n, nz or n, bc)
    return raw, core.expand(*raw)


def relerr(got, want):
    """tests/acceptance.cpp:28-30 — Frobenius relative error."""
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def max_slice_relerr(got, want):
    """max over elements of ||x_gpu - x_oracle||_F / ||x_oracle||_F."""
    got = np.asarray(got).reshape(got.shape[0], -1)
    want = np.asarray(want).reshape(want.shape[0], -1)
    num = np.linalg.norm(got - want, axis=1)
    den = np.maximum(np.linalg.norm(want, axis=1), 1e-300)
    return float(np.max(num / den))


def solve_skeleton(em, colptr, rowidx, vals, b, ubdry, d2):
    """global_system.cpp:106-165 restated with scipy (SuperLU) for the free block."""
    ndof = len(b)
    H = sp.csc_matrix((vals, rowidx, colptr), shape=(ndof, ndof))
    fixed = np.zeros(ndof, dtype=bool)
    uhat = np.zeros(ndof)
    dirf = np.asarray(em.dirfaces)
    for j, f in enumerate(dirf):
        fixed[f * d2:(f + 1) * d2] = True
        uhat[f * d2:(f + 1) * d2] = ubdry[j * d2:(j + 1) * d2]
    free = np.flatnonzero(~fixed)
    Hff = H[free][:, free].tocsc()
    rhs = b[free] - H[free][:, np.flatnonzero(fixed)] @ uhat[fixed]
    uhat[free] = spla.spsolve(Hff, rhs)
    return uhat


def solve_level(raw, k, prob: Problem, tau=1.0, quad_bump=0, threads=1, errors=True):
    """study.cpp:10-43 through the oracle; returns a dict of intermediates."""
    em = core.expand(*raw)
    qd = 2 * k + 2 + quad_bump
    t = core.tables(k, qd, qd)
    nelt = em.n_elements
    tauf = core.Stabilization(np.full((nelt, 4), float(tau)))
    kap, c, f, u = field(prob.kappa), field(prob.c), field(prob.f), field(prob.u)
    q = vfield(prob.q)
    ms = core.build_element_matrices(em, t, kap, c, f, tauf)
    lb = core.local_blocks(ms)
    C, Cf = core.condense(lb, threads)
    colptr, rowidx, vals, b = core.assemble(em, C, Cf)
    b = b - core.neumann_load(em, k, qd, q)
    ub = core.dirichlet_project(em, k, qd, u)
    d2 = (k + 1) * (k + 2) // 2
    uhat = solve_skeleton(em, colptr, rowidx, vals, b, ub, d2)
    qx, qy, qz, uu = core.local_recover(lb, core.gather_traces(em, d2, uhat), threads)
    t1 = core.tables(k + 1, 2 * (k + 1) + 2 + quad_bump, qd)
    ustar = core.postprocess_star(em, t1, kap, qx, qy, qz, uu)
    out = dict(em=em, t=t, ms=ms, lb=lb, C=C, Cf=Cf, H=(colptr, rowidx, vals), b=b, ub=ub,
               uhat=uhat, q=(qx, qy, qz), u=uu, ustar=ustar, tau=tauf)
    if errors:
        out["errors"] = core.compute_errors(em, ms, tauf, u, q, k, uhat, qx, qy, qz, uu, ustar)
    return out
