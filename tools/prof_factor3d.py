"""Developer profile driver: device factorization of C5-size 3D subdomains (57^3 local grids:
n = 32 * HS_P intervals per axis, HS_P^3 subdomains, 12-cell PML), omega = 2 pi 12."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_02585_b200 as hs
p = int(os.environ.get("HS_P", "2"))
t = time.perf_counter()
s = hs.DdmSolver(hs.ProblemSetup(3, [32 * p] * 3, [p] * 3, hs.Medium("constant", kappa=2 * math.pi * 12), pml_width=12))
print(f"{p}^3 subdomains of 57^3: setup {time.perf_counter() - t:.2f} s, factor_seconds {s.factor_seconds():.2f}, "
      f"device factorization {s.sub_stats(0).factor_seconds:.2f} s", flush=True)
