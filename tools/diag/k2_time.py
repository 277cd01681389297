"""Time K2 (node build) on a config's mesh for several field sets:
k2_time.py LIB CONFIG. Separates the field-evaluation share of K2 from the
node GEMM (constant fields leave only the GEMM and the stores)."""
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
p = cfg.problem
sets = {"config": (p.kappa, p.c, p.f), "const": ("1.5", "1.0", "1.0"),
        "kappa only": (p.kappa, "1.0", "1.0"), "f only": ("1.5", "1.0", p.f)}
for name, (kap, c, f) in sets.items():
    tb = []
    for i in range(8):
        eng.build_condense(g, kap, c, f)
        torch.cuda.synchronize()
        if i >= 2:
            tb.append(eng.stage_times()["node_build"])
    print(f"{cfg.name} {name:>10}: node build median {np.median(tb):.3f} ms")
