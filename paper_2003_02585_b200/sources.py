"""Seeded synthetic right-hand sides for the BASELINE workloads (host-side input producer).

SURVEY.md §8(d): the reference's Gaussian SourceSpec ties its width to kappa
(src/harness.cpp:107-124), so the benchmark harness builds
``f(x) = exp(-|x - x_s|^2 / (2 sigma^2))`` with sigma = 2h on interior (non-PML) nodes — the
same inside-mask as src/harness.cpp:116-122 — and locations from ``std::mt19937_64(seed)`` with
``u = (rng() >> 11) * 2^-53`` per axis. Both the GPU path and the reference CPU baseline are fed
the same ``b = DdmSolver::scale_source(f)``.
"""
from __future__ import annotations

import numpy as np

_MASK = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the engine the reference seeds its shot sources with)."""

    def __init__(self, seed=5489):
        mt = [0] * 312
        mt[0] = seed & _MASK
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK
        self.mt, self.idx = mt, 312

    def __call__(self):
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK

    def unit(self):
        return (self() >> 11) * (1.0 / 9007199254740992.0)


def seeded_centers(seed, count, dim, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
    rng = MT19937_64(seed)
    return [[lo[a] + rng.unit() * (hi[a] - lo[a]) for a in range(dim)] for _ in range(count)]


def gaussian_sources(dim, glo, ghi, h, origin, centers, sigma, interior_lo=(0.0,) * 3, interior_hi=(1.0,) * 3):
    """f for each centre on the padded global grid [glo, ghi] (axis 0 fastest), RHS-major
    (len(centers), N) complex128."""
    sizes = [ghi[a] - glo[a] + 1 for a in range(dim)]
    axes = [origin[a] + (glo[a] + np.arange(sizes[a])) * h[a] for a in range(dim)]
    inside = [(x >= interior_lo[a]) & (x <= interior_hi[a]) for a, x in enumerate(axes)]
    out = np.zeros((len(centers), int(np.prod(sizes))), dtype=np.complex128)
    for r, c in enumerate(centers):
        # separable: exp(-sum_a (x_a - c_a)^2 / 2s^2) with the same per-node r2 summation order
        d2 = [(x - c[a]) * (x - c[a]) for a, x in enumerate(axes)]
        if dim == 2:
            r2 = d2[0][None, :] + d2[1][:, None]
            m = inside[0][None, :] & inside[1][:, None]
        else:
            r2 = (d2[0][None, None, :] + d2[1][None, :, None]) + d2[2][:, None, None]
            m = inside[0][None, None, :] & inside[1][None, :, None] & inside[2][:, None, None]
        out[r] = np.where(m, np.exp(-r2 / (2.0 * sigma * sigma)), 0.0).ravel()
    return out


def gaussian_random_velocity(n, seed, corr_len=0.05, lo=0.0, hi=1.0, dtype=np.float32):
    """BASELINE config 4's smooth heterogeneous medium on an (n+1)^2 node lattice over [lo, hi]^2
    (axis 0 fastest, the HSVG sample order, include/helmsweep/media.hpp:22-27):
    c = 1 + 0.5 (1 + tanh g) / 2, g a seeded stationary Gaussian field with Gaussian covariance
    exp(-|r|^2 / (2 corr_len^2)), unit variance. g is white noise filtered in Fourier space by the
    square root of the covariance's spectral density, exp(-|k|^2 corr_len^2 / 4) (periodic
    synthesis on a lattice padded by 4 correlation lengths, then cropped), and normalised to zero
    mean and unit variance. The reference defines no generator; this one is archived with its
    seed so both paths read the same file."""
    m = n + 1
    h = (hi - lo) / n
    pad = int(np.ceil(4 * corr_len / h))
    M = m + pad
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((M, M))
    k = 2 * np.pi * np.fft.fftfreq(M, d=h)
    k2 = k[:, None] ** 2 + k[None, :] ** 2
    g = np.fft.ifft2(np.fft.fft2(w) * np.exp(-k2 * corr_len ** 2 / 4)).real[:m, :m]
    g = (g - g.mean()) / g.std()
    c = 1.0 + 0.5 * (1.0 + np.tanh(g)) / 2.0
    return np.ascontiguousarray(c.T, dtype=dtype)  # [y][x] rows -> axis 0 (x) fastest when flattened
