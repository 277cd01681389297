"""Skeleton solve on the GPU at a BASELINE config: iterations, time, residual."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1305_1489_b200.configs import CONFIGS  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
prob = cfg.problem
mesh = HostMesh.box(cfg.n, bc=prob.bc, perturb=cfg.perturb, seed=cfg.seed)
eng = Engine(0)
eng.set_degree(cfg.k)
dm = eng.upload(mesh)
g = eng.geometry(dm, cfg.tau)
cs = eng.build_condense(g, prob.kappa, prob.c, prob.f)
pat = eng.pattern_device(dm)
sys_ = eng.assemble(dm, pat, cs)
ub = eng.dirichlet_project(dm, prob.u)
eng.neumann_load(dm, g, prob.q, b=sys_.b, alpha=-1.0)
torch.cuda.synchronize()
for rtol in (1e-8, 1e-13, 1e-13, 1e-13):
    t0 = time.perf_counter()
    uhat, info = eng.solve_skeleton(dm, pat, sys_, ub, rtol=rtol)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ms = 1e3 * (t1 - t0)
    print(f"{cfg.name}: ndof {sys_.b.numel()} nnz {sys_.vals.numel()} rtol {rtol:g}: {info['iterations']} it, "
          f"{ms:.1f} ms ({ms / max(info['iterations'], 1):.3f} ms/it), relres {info['relres']:.2e}")
