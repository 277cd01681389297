"""Time K7 (convection_bilinear_matrices) on C4's mesh with the config's
program beta and with constant beta: k7_time.py [LIB]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1305_1489_b200 import _lib as L  # noqa: E402

if len(sys.argv) > 1:
    L.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402
from paper_1305_1489_b200.configs import CONFIGS  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh  # noqa: E402

cfg = CONFIGS["C4"]
mesh = HostMesh.box(cfg.n, bc=cfg.problem.bc)
eng = Engine(0)
eng.set_degree(cfg.k)
dm = eng.upload(mesh)
g = eng.geometry(dm, 1.0)
out = None
for label, beta in (("program", cfg.upwind_beta), ("const", ("0.3", "0.2", "0.5"))):
    ts = []
    for i in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        eng.convection_bilinear_matrices(g, beta)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"K7 C4 beta={label} {beta}: {sorted(ts[2:])[len(ts[2:]) // 2]:.3f} ms")
