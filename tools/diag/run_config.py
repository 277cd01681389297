"""One pass of a config's pipeline at full size (for ncu captures of a single
kernel, e.g. ncu -k regex:condense6 -c 1 python tools/diag/run_config.py C4):
geometry (+ upwind tau), build+condense, recover, then per config the
postprocess (C5), the convection block (C4), and the face-ordered scatter."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1305_1489_b200.configs import CONFIGS  # noqa: E402
from paper_1305_1489_b200.engine import Engine, Field, HostMesh, dim2  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
what = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else {"all"}
p = cfg.problem
mesh = HostMesh.box(cfg.n, bc=p.bc, perturb=cfg.perturb, seed=cfg.seed)
eng = Engine(0)
eng.set_degree(cfg.k)
dm = eng.upload(mesh)
g = eng.geometry(dm, 1.0)
tau = eng.upwind_tau(g, cfg.upwind_beta) if cfg.upwind_beta else cfg.tau
g = eng.geometry(dm, tau)
kap, cc, ff = Field.program(p.kappa), Field.program(p.c), Field.program(p.f)
cs = eng.build_condense(g, kap, cc, ff)
d2 = dim2(cfg.k)
uhat = torch.sin(torch.arange(dm.nfc * d2, dtype=torch.float64, device="cuda") * 0.013)
ls = eng.recover(g, dm, cs, uhat)
if cfg.postprocess and ("all" in what or "post" in what):
    eng.set_postprocess_rule()
    eng.postprocess_star(g, kap, ls)
if cfg.upwind_beta and ("all" in what or "conv" in what):
    eng.convection_bilinear_matrices(g, cfg.upwind_beta)
if "all" in what or "scatter" in what:
    pat = eng.pattern(mesh)
    eng.assemble(dm, pat, cs)
torch.cuda.synchronize()
print("ran", cfg.name, sorted(what))
