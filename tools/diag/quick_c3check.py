import sys, os
sys.path[:0]=['/root/repo','/root/repo/tests']
from paper_1305_1489_b200 import _lib as L
L.LIB_PATH=os.path.abspath(sys.argv[1])
import numpy as np
from gpu_util import gpu_pipeline, oracle_condense, oracle_mesh, np_
from oracle_util import max_slice_relerr
from paper_1305_1489_b200.engine import HostMesh
KAP = "2 + sin(x)*sin(y)*sin(z)"; CC = "1 + 0.5*(x*x + y*y + z*z)"; FF = "cos(x + 2*y - z)"
mesh = HostMesh.box(2, bc="dirichlet_x")
eng, dm, g, cs = gpu_pipeline(mesh, 3, KAP, CC, FF)
_, _, lb, C, Cf = oracle_condense(oracle_mesh(mesh), 3, KAP, CC, FF, 1.0)
e = np.linalg.norm((np_(cs.C_slices())-C).reshape(48,-1),axis=1)/np.linalg.norm(C.reshape(48,-1),axis=1)
print(os.path.basename(sys.argv[1]), "C err max", e.max(), "bad elements", np.nonzero(e>1e-10)[0][:20], "Cf", max_slice_relerr(np_(cs.Cf_cols()), Cf.T))
# cache Vs vs numpy for the first bad element
K = int(np.argmax(e))
d3, m = 20, 40
ns = d3 * (d3 + 1) // 2
F = np_(cs.factors.view(dm.nelt, -1))[K]
Vs = F[ns:ns + d3 * m].reshape(m, d3).T
A1 = lb.A1[K]; M = A1[:d3, :d3]; Cb = A1[3 * d3:, :3 * d3]; D = A1[3 * d3:, 3 * d3:]
Mbi = np.kron(np.eye(3), np.linalg.inv(M)); S = D + Cb @ Mbi @ Cb.T
E = lb.A3[K][:, :3 * d3]; tDP = lb.A3[K][:, 3 * d3:]; V = Cb @ Mbi @ E.T + tDP.T
Vs_ref = np.linalg.solve(S, V)
err = np.abs(Vs - Vs_ref) / np.abs(Vs_ref).max()
print("element", K, "Vs err by row", np.round(err.max(axis=1), 3))
print("Vs err by col tile", [round(err[:, 8*j:8*j+8].max(), 3) for j in range(5)])
Cg = np_(cs.C_slices())[K]
D = np.abs(Cg - C[K]) / np.abs(C[K]).max()
print("C err by (row tile, col tile):")
print(np.array([[round(D[8*i:8*i+8, 8*j:8*j+8].max(), 4) for j in range(5)] for i in range(5)]))
