"""Native NCCL transport (hs_ddm_create_nccl) on one GPU: world 1 runs the partitioned machinery
(ownership, home-node accumulation, NCCL reductions on the solver stream, graph capture) and must
reproduce the plain solver bit for bit. Multi-rank NCCL needs one GPU per rank (a gpurun box has
one); the multi-rank exchange logic is covered by the gloo tests (tests/test_partition.py)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_client_nccl_world1(tmp_path):
    """A C++ client of include/helmsweep_b200.h drives the native NCCL path (world 1)."""
    lib = os.path.join(ROOT, "paper_2003_02585_b200")
    exe = str(tmp_path / "nccl_world1")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "nccl_world1.cpp"), "-L", lib, "-lhelmsweep_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "ok:" in r.stdout


def test_python_nccl_world1_matches_golden(golden):
    import ast
    import paper_2003_02585_b200 as hs
    from paper_2003_02585_b200 import multi
    z = golden("ddm_2d_layered")
    med = ast.literal_eval(str(z["medium"]))
    m = hs.Medium("two_layered", kappa_down=med["media.kappa_down"], kappa_up=med["media.kappa_up"],
                  axis=med["media.axis"], eta=med["media.eta_L"], eps=med["media.epsilon"])
    setup = hs.ProblemSetup(2, [int(z["n"])] * 2, list(z["parts"]), m, pml_width=int(z["pad"]))
    s = multi.NcclDdmSolver(setup, 0, 0, 1, multi.nccl_unique_id())
    plain = hs.DdmSolver(setup)
    rounds = int(z["rounds"])
    U = s.ddm_solve(z["b"], rounds, None, True)
    assert np.array_equal(U, plain.ddm_solve(z["b"], rounds, None, True))
    for r in range(U.shape[0]):
        assert np.linalg.norm(U[r] - z["u"][r]) / np.linalg.norm(z["u"][r]) <= 1e-9
