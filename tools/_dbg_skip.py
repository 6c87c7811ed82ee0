import sys, os, ast
sys.path.insert(0, '.')
import numpy as np
import paper_2003_02585_b200 as hs
z = np.load('tests/golden/ddm_2d_2x2.npz')
med = ast.literal_eval(str(z["medium"]))
s = hs.DdmSolver(hs.ProblemSetup(2, [int(z["n"])] * 2, list(z["parts"]), hs.Medium("constant", kappa=med["media.kappa"]), pml_width=int(z["pad"])))
for r in range(2):
    reps = []
    U = s.ddm_solve(z["b"][r], int(z["rounds"]), reps, True)
    print(os.environ.get("HS_NO_FRONT_SKIP"), r, np.linalg.norm(U - z["u"][r]) / np.linalg.norm(z["u"][r]), reps[0].sweep_contrib_norm, list(z["contrib_norm"][r]))
