"""Time K6 (postprocess_star) of a libhdg_b200 build on a config's mesh:
post_time.py LIB CONFIG (random q, u: values do not change the cost)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1305_1489_b200 import _lib as L  # noqa: E402

L.LIB_PATH = os.path.abspath(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1305_1489_b200.configs import CONFIGS  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh, LocalSolution, dim3  # noqa: E402

cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C5"]
mesh = HostMesh.box(cfg.n, bc=cfg.problem.bc, perturb=cfg.perturb, seed=cfg.seed)
eng = Engine(0)
eng.set_degree(cfg.k)
eng.set_postprocess_rule()
dm = eng.upload(mesh)
g = eng.geometry(dm, cfg.tau)
d3 = dim3(cfg.k)
ls = LocalSolution(*(torch.randn(dm.nelt, d3, dtype=torch.float64, device="cuda") for _ in range(4)))
ts = []
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    us = eng.postprocess_star(g, cfg.problem.kappa, ls)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
print(f"{os.path.basename(sys.argv[1])} {cfg.name}: postprocess median {np.median(ts):.3f} ms")
