import sys, torch
sys.path.insert(0, '/root/repo')
from paper_1305_1489_b200.configs import CONFIGS
from paper_1305_1489_b200.engine import Engine, Field, HostMesh, dim2
cfg = CONFIGS["C5"]; p = cfg.problem
mesh = HostMesh.box(8, bc=p.bc)
eng = Engine(0); eng.set_degree(cfg.k); dm = eng.upload(mesh); g = eng.geometry(dm, cfg.tau)
kap = Field.program(p.kappa)
cs = eng.build_condense(g, kap, Field.program(p.c), Field.program(p.f))
uhat = torch.sin(torch.arange(dm.nfc * dim2(cfg.k), dtype=torch.float64, device="cuda") * 0.013)
ls = eng.recover(g, dm, cs, uhat)
eng.set_postprocess_rule()
print("before:", repr(eng.jit_status))
eng.postprocess_star(g, kap, ls)
torch.cuda.synchronize()
print("after post:", repr(eng.jit_status))
