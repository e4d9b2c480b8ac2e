"""Seeded synthetic inputs with the shapes and value distributions of
BASELINE.json's configs.  No dataset exists for this path;
these generators stand in for the reference's own analytic test problems.

configs[1]: domain [0,1)^3, node-based x_i = i/n (as Grid2D, pde.cpp:16-19),
a = 1 + 0.5 sin(2 pi x) cos(2 pi y) sin(2 pi z), U = sum of 16 seeded Fourier
modes with integer wavevectors 1 <= |k| <= 8, amplitude U[0,1), phase U[0,2pi).
Works on numpy (host) or torch (device) arrays.
"""
from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi


def modes(seed: int = 1309, count: int = 16, kmax: float = 8.0):
    """Integer wavevectors (rejection sampled), amplitudes, phases."""
    rng = np.random.default_rng(seed)
    ks, amps, phases = [], [], []
    while len(ks) < count:
        k = rng.integers(-8, 9, size=3)
        nk = float(np.sqrt((k * k).sum()))
        if 1.0 <= nk <= kmax:
            ks.append(k.astype(np.float64))
            amps.append(rng.random())
            phases.append(rng.random() * TWO_PI)
    return np.array(ks), np.array(amps), np.array(phases)


def _grid(n, xp, device=None):
    if xp is np:
        x = np.arange(n, dtype=np.float64) / n
        return x[None, None, :], x[None, :, None], x[:, None, None]
    x = xp.arange(n, dtype=xp.float64, device=device) / n
    return x.view(1, 1, n), x.view(1, n, 1), x.view(n, 1, 1)


def narrow3d_inputs(n: int, seed: int = 1309, xp=np, device=None):
    """(a, U) of shape (n, n, n), x fastest."""
    x, y, z = _grid(n, xp, device)
    s = xp.sin
    c = xp.cos
    a = 1.0 + 0.5 * s(TWO_PI * x) * c(TWO_PI * y) * s(TWO_PI * z)
    ks, amps, ph = modes(seed)
    u = xp.zeros((n, n, n), dtype=xp.float64) if xp is np else \
        xp.zeros((n, n, n), dtype=xp.float64, device=device)
    for k, A, p in zip(ks, amps, ph):
        u = u + A * s(TWO_PI * (k[0] * x + k[1] * y + k[2] * z) + p)
    if xp is np:
        return np.ascontiguousarray(a), np.ascontiguousarray(u)
    return a.contiguous(), u.contiguous()


def narrow3d_exact(n: int, seed: int = 1309, xp=np, device=None):
    """Analytic div(a grad U) = grad a . grad U + a lap U on the nodes."""
    x, y, z = _grid(n, xp, device)
    s, c = xp.sin, xp.cos
    a = 1.0 + 0.5 * s(TWO_PI * x) * c(TWO_PI * y) * s(TWO_PI * z)
    ax = 0.5 * TWO_PI * c(TWO_PI * x) * c(TWO_PI * y) * s(TWO_PI * z)
    ay = -0.5 * TWO_PI * s(TWO_PI * x) * s(TWO_PI * y) * s(TWO_PI * z)
    az = 0.5 * TWO_PI * s(TWO_PI * x) * c(TWO_PI * y) * c(TWO_PI * z)
    ks, amps, ph = modes(seed)
    out = 0.0
    for k, A, p in zip(ks, amps, ph):
        th = TWO_PI * (k[0] * x + k[1] * y + k[2] * z) + p
        g = A * TWO_PI * c(th)
        out = out + ax * g * k[0] + ay * g * k[1] + az * g * k[2] \
            - a * (A * TWO_PI ** 2 * float(k @ k)) * s(th)
    return out


# --------------------------------------------------------------------------
# NS states (configs[0], [2], [3], [4]); primitive fields on a periodic
# n^3 box of spacing dx: T [K], p [Pa], velocity [m/s], mass fractions.
NSP = 9
SP = dict(H2=0, O2=1, H2O=2, H=3, O=4, OH=5, HO2=6, H2O2=7, N2=8)


def _smooth_modes(rng, count, kmax):
    ks, ph = [], []
    while len(ks) < count:
        k = rng.integers(-kmax, kmax + 1, size=3)
        if 0 < (k * k).sum() <= kmax * kmax:
            ks.append(k.astype(np.float64))
            ph.append(rng.random() * TWO_PI)
    return ks, ph


def ns_primitives(n: int, seed: int = 1309, hot_spot: bool = False, ignition: bool = False,
                  ny: int = None, nz: int = None, z0: int = 0, nz_global: int = None):
    """configs[0] generator: T = 1200 K + 300 K x (sum of 4 random-phase
    sinusoids, normalised), p = 1 atm, velocity = 8 random Fourier modes of
    amplitude 10 m/s, Y = smooth seeded H2/O2/N2 blend + 1e-6 radicals,
    normalised.  hot_spot: Gaussian T bump to 1800 K, radius 20 cells
    (configs[3]).  ignition: 600 K stoichiometric H2/air with a 1500 K
    Gaussian kernel (configs[4]).  ny/nz/z0/nz_global select a z-slab of a
    larger periodic box (multi-GPU)."""
    ny = ny or n
    nz = nz or n
    nzg = nz_global or nz
    rng = np.random.default_rng(seed)
    i = np.arange(n, dtype=np.float64)[None, None, :] / n
    j = np.arange(ny, dtype=np.float64)[None, :, None] / ny
    kz = ((z0 + np.arange(nz)) % nzg).astype(np.float64)[:, None, None] / nzg

    def field(ks, ph):
        out = np.zeros((nz, ny, n))
        for k, p_ in zip(ks, ph):
            out = out + np.sin(TWO_PI * (k[0] * i + k[1] * j + k[2] * kz) + p_)
        return out

    ks, ph = _smooth_modes(rng, 4, 2)
    sT = field(ks, ph)
    T = 1200.0 + 300.0 * sT / 4.0  # |sum of 4 unit sinusoids| <= 4
    u = []
    for _ in range(3):
        ks, ph = _smooth_modes(rng, 8, 2)
        s = field(ks, ph)
        u.append(10.0 * s / 8.0)
    ks, ph = _smooth_modes(rng, 2, 1)
    s1 = field(ks, ph)
    ks, ph = _smooth_modes(rng, 2, 1)
    s2 = field(ks, ph)
    Y = np.zeros((NSP, nz, ny, n))
    Y[SP["H2"]] = 0.02 + 0.01 * (s1 / 2.0)
    Y[SP["O2"]] = 0.22 + 0.02 * (s2 / 2.0)
    for sp in ("H2O", "H", "O", "OH", "HO2", "H2O2"):
        Y[SP[sp]] = 1e-6
    if ignition:
        T = np.full((nz, ny, n), 600.0)
        Y[SP["H2"]] = 0.0285
        Y[SP["O2"]] = 0.2264
    if hot_spot or ignition:
        c = np.array([n / 2.0, ny / 2.0, nzg / 2.0])

        def pdist(a, L):
            d = np.abs(a - 0.0)
            return np.minimum(d, L - d)
        xi = np.arange(n, dtype=np.float64)[None, None, :]
        yj = np.arange(ny, dtype=np.float64)[None, :, None]
        zk = ((z0 + np.arange(nz)) % nzg).astype(np.float64)[:, None, None]
        r2 = pdist(xi - c[0], n) ** 2 + pdist(yj - c[1], ny) ** 2 + pdist(zk - c[2], nzg) ** 2
        g = np.exp(-r2 / 20.0 ** 2)
        peak = 1500.0 if ignition else 1800.0
        T = T + (peak - T) * g
    Y[SP["N2"]] = 1.0 - Y[:SP["N2"]].sum(axis=0)
    Y = Y / Y.sum(axis=0)
    p = np.full((nz, ny, n), 101325.0)
    return (np.ascontiguousarray(T), np.ascontiguousarray(p),
            np.ascontiguousarray(np.stack(u)), np.ascontiguousarray(Y))
