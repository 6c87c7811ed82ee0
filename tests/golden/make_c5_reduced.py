"""Golden fixture for BASELINE config 5 at its own subdomain size, produced by the REFERENCE
(oracle/_ref, compiled in place from /root/reference). Run in the build container:

    python tests/golden/make_c5_reduced.py

C5 is 3D, 128^3 + 12-cell PML, 4x4x4 subdomains, omega = 2 pi 12 (h = 1/128). Its factors do not
fit this host's RAM in the reference's m x k storage, so SURVEY.md §8(d) asks for parity on a
reduced geometry with the SAME subdomain size: interior [0, 0.5]^3 with grid.n = 64 (h = 1/128),
2x2x2 subdomains -> owned 33^3 + 2x12 PML = 57^3 local grids (185 193 nodes, fronts up to
m = 4845, k = 3249 -- exactly C5's), kappa = 2 pi 12, one round of 8 sweeps, one seeded Gaussian
source (sigma = 2h). Stores u, the SolveReport counters, contribution norms, round residuals,
per-subdomain factor_nnz / peak_bytes, and the SHA-256 of b (the GPU test rebuilds b itself).
"""
from __future__ import annotations

import hashlib
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import hs_oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

COUNTERS = ["traces_generated", "traces_routed", "traces_discarded", "local_solves", "skipped_zero_solves"]
CFG = {"dim": 3, "grid.n": [64, 64, 64], "partition": [2, 2, 2], "pml.width": 12,
       "interior.lo": [0.0, 0.0, 0.0], "interior.hi": [0.5, 0.5, 0.5],
       "media.kind": "constant", "media.kappa": 2 * math.pi * 12}
SEED = 5000


def main():
    t = time.time()
    s = R.RefSolver(CFG, 4)  # 4 workers: a 57^3 factorization holds ~8 GB of dense fronts at its peak
    print("factorization", time.time() - t, "s", flush=True)
    interior = O.Box(3, (0.0, 0.0, 0.0), (0.5, 0.5, 0.5))
    centers = O.seeded_centers(SEED, 1, interior)
    ggrid = O.LocalGrid(3, O.GridRange(3, s.lo, s.hi), s.hgrid, s.origin)
    f = O.gaussian_source(ggrid, interior, centers, 2.0 / 128)
    b = s.scale_source(f[:, 0].copy())
    t = time.time()
    u, rep = s.ddm_solve(b, 1, True)
    print("ddm_solve", time.time() - t, "s", flush=True)
    np.savez_compressed(
        os.path.join(HERE, "ddm_3d_c5_reduced.npz"), cfg=repr(CFG), centers=np.array(centers), sigma=2.0 / 128,
        b_sha256=hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest(), u=u,
        counters=np.array([rep[k] for k in COUNTERS]), contrib_norm=np.array(rep["sweep_contrib_norm"]),
        round_residuals=np.array(rep["round_residuals"]), ref_factor_seconds=s.factor_seconds,
        factor_nnz=np.array([s.sub_info(i)["factor_nnz"] for i in range(s.nsub)]),
        peak_bytes=np.array([s.sub_info(i)["peak_bytes"] for i in range(s.nsub)]),
        lo=np.array(s.lo), hi=np.array(s.hi))


if __name__ == "__main__":
    main()
