"""Setup-path timing: host expand + pattern (C++) vs the device pipeline, on a
box of n^3 cells (default 64 = C5)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1305_1489_b200.engine import Engine, HostMesh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mesh = HostMesh.box(n, bc="dirichlet_x")
X, E, D, N = mesh.coordinates, mesh.elements, mesh.dirichlet, mesh.neumann
t0 = time.perf_counter()
m2 = HostMesh.from_raw(X, E, D, N)
t1 = time.perf_counter()
fb, nb, sl = m2.pattern()
t2 = time.perf_counter()
eng = Engine(0)
eng.set_degree(3)
Xd, Ed = torch.from_numpy(X).cuda(), torch.from_numpy(E).cuda()
Dd, Nd = torch.from_numpy(D).cuda(), torch.from_numpy(N).cuda()
for i in range(3):
    torch.cuda.synchronize()
    s0 = time.perf_counter()
    dm = eng.expand(Xd, Ed, Dd, Nd)
    torch.cuda.synchronize()
    s1 = time.perf_counter()
    p = eng.pattern_device(dm, csr=False)
    torch.cuda.synchronize()
    s2 = time.perf_counter()
print(f"n={n} nelt={m2.n_elements} nfc={m2.n_faces}: host expand {1e3*(t1-t0):.1f} ms, host pattern "
      f"{1e3*(t2-t1):.1f} ms | device expand {1e3*(s1-s0):.2f} ms, device pattern {1e3*(s2-s1):.2f} ms")
