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
