import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2108_13229_b200 import sdc
g = dict(np.load("tests/golden/system_n16.npz"))
n = int(g["n_total"])
A = sdc.SparseMatrix(n, n, g["A_rowptr"], g["A_col"], g["A_val"])
s = sdc.CoupledSystem(A, g["rhs"], int(g["n"]), int(g["n_u"]), int(g["n_vel"]), int(g["n_pff"]), int(g["n_ppm"]))
try:
    p = sdc.TdPreconditioner(s, "td_bgs")
    print("ok omega", p.omega(), g["omega"])
    z = p.apply(g["apply_r"]); print("rel", np.linalg.norm(z-g["apply_z"])/np.linalg.norm(g["apply_z"]))
except Exception as e:
    print("ERR", e)
