"""Time K3 (build_condense) and K5 (recover) of a libhdg_b200 variant:
sweep_time.py LIB CONFIG."""
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
eng.set_timing(True)
ts, tr, tb = [], [], []
d2 = (cfg.k + 1) * (cfg.k + 2) // 2
uhat = torch.sin(torch.arange(dm.nfc * d2, dtype=torch.float64, device="cuda") * 0.37)
for i in range(8):
    cs = eng.build_condense(g, cfg.problem.kappa, cfg.problem.c, cfg.problem.f)
    ls = eng.recover(g, dm, cs, uhat)
    torch.cuda.synchronize()
    st = eng.stage_times()
    if i >= 2:
        ts.append(st["condense"])
        tb.append(st["node_build"])
        tr.append(st["recover"])
print(f"{os.path.basename(sys.argv[1])} {cfg.name}: node build median {np.median(tb):.3f} ms  "
      f"condense median {np.median(ts):.3f} ms  "
      f"recover median {np.median(tr):.3f} ms")
