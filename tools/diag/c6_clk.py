"""Per-phase clocks of K3 v6 (a -DHDG_C6_CLK build writes them into Cf):
c6_clk.py LIB CONFIG -> median cycles per element of derive+mib / Y,S,V^T
loop / prefetch / S sweep / C phase / next M sweep."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1305_1489_b200 import _lib as L  # noqa: E402

L.LIB_PATH = os.path.abspath(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1305_1489_b200.configs import CONFIGS  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh  # noqa: E402

cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C2"]
mesh = HostMesh.box(cfg.n, bc=cfg.problem.bc, perturb=cfg.perturb, seed=cfg.seed)
eng = Engine(0)
eng.set_degree(cfg.k)
dm = eng.upload(mesh)
g = eng.geometry(dm, cfg.tau)
for _ in range(2):
    cs = eng.build_condense(g, cfg.problem.kappa, cfg.problem.c, cfg.problem.f)
torch.cuda.synchronize()
cf = cs.Cf_cols().cpu().numpy() if hasattr(cs, "Cf_cols") else None
m = cf.shape[0]
clk = cf[:5, :].T if cf.shape[0] < cf.shape[1] else cf[:, :5]
med = np.median(clk[1:-1000], axis=0)
names = ["derive+mib", "Y/S/VT loop", "S sweep+sib+fs", "C phase", "next M sweep"]
print(os.path.basename(sys.argv[1]), cfg.name, " ".join(f"{n} {v:.0f}" for n, v in zip(names, med)), f"sum {med.sum():.0f}")
