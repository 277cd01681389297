import sys, os
sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo')
from paper_1305_1489_b200 import _lib as L
L.LIB_PATH = os.path.abspath(sys.argv[1])
from gpu_util import gpu_pipeline, np_, oracle_condense, oracle_mesh
from oracle_util import max_slice_relerr
from paper_1305_1489_b200.engine import HostMesh
KAP = "2 + sin(x)*sin(y)*sin(z)"; CC = "1 + 0.5*(x*x + y*y + z*z)"; FF = "cos(x + 2*y - z)"
for k, n, bc in [(4, 1, "dirichlet_top_bottom"), (5, 1, "dirichlet_top_bottom"), (4, 2, "dirichlet_x")]:
    mesh = HostMesh.box(n, bc=bc)
    em = oracle_mesh(mesh)
    eng, dm, g, cs = gpu_pipeline(mesh, k, KAP, CC, FF)
    _, _, _, C, Cf = oracle_condense(em, k, KAP, CC, FF, 1.0)
    print(os.path.basename(sys.argv[1]), k, n, "C", max_slice_relerr(np_(cs.C_slices()), C), "Cf", max_slice_relerr(np_(cs.Cf_cols()), Cf.T))
