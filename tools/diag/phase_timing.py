"""Diagnostics: per-phase cycle counts of the CTA-batched condensation kernel
(build with -DHDG_PHASE_TIMING, e.g. tools/diag/sweep_build.sh "pt,-DHDG_PHASE_TIMING"):
phase_timing.py CONFIG [LIB]."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1305_1489_b200 import _lib as L  # noqa: E402

L.LIB_PATH = os.path.abspath(sys.argv[2]) if len(sys.argv) > 2 else os.path.join(ROOT, "tools", "diag", "libhdg_b200_phase.so")
lib = L.lib()
lib.hdg_b200_debug_phase_clocks.argtypes = [C.c_void_p]
import torch  # noqa: E402
from paper_1305_1489_b200.configs import CONFIGS  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
mesh = HostMesh.box(cfg.n, bc=cfg.problem.bc, perturb=cfg.perturb, seed=cfg.seed)
eng = Engine(0)
eng.set_degree(cfg.k)
dm = eng.upload(mesh)
g = eng.geometry(dm, cfg.tau)
for _ in range(3):
    cs = eng.build_condense(g, cfg.problem.kappa, cfg.problem.c, cfg.problem.f)
torch.cuda.synchronize()
out = np.zeros((148, 8, 8), dtype=np.int64)
L.check(lib.hdg_b200_debug_phase_clocks(out.ctypes.data))
d = np.diff(out[:, 1:7, :6], axis=2)  # batches 1..6, phases P1..P5
names = ["P1 Zp+R", "P2 S+V", "P3 GJ+WZp", "P4 Vs", "P5 C"]
tot = d.sum(axis=2)
print(f"{cfg.name}: median cycles per batch {np.median(tot):.0f}")
for i, n in enumerate(names):
    print(f"  {n:10s} median {np.median(d[:, :, i]):7.0f}  p90 {np.percentile(d[:, :, i], 90):7.0f}")
