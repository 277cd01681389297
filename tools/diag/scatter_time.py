"""K4 scatter timing of a libhdg_b200 build: scatter_time.py LIB [CONFIG]."""
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
cs = eng.build_condense(g, cfg.problem.kappa, cfg.problem.c, cfg.problem.f)
pat = eng.pattern_device(dm)
sysH = eng.assemble(dm, pat, cs)
eng.set_timing(True)
ts = []
for i in range(8):
    eng.assemble(dm, pat, cs, out=sysH)
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(eng.stage_times()["scatter"])
    else:
        eng.stage_times()
m = 4 * (cfg.k + 1) * (cfg.k + 2) // 2
gb = 2 * 8.0 * m * (m + 1) * dm.nelt / 1e9
print(f"{os.path.basename(sys.argv[1])} {cfg.name}: scatter median {np.median(ts):.3f} ms = {gb / np.median(ts):.0f} GB/s")
