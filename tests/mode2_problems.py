"""Test problems for MRSDC mode 2 / the backward-Euler Newton (f1 implicit).

Each problem is stated once as array code and evaluated either with numpy
(the oracle / reference callbacks) or with torch on the device (the GPU
path); both evaluate the same elementwise IEEE operations in the same
order, so the two sides see identical f values.

  oscillator(sigma)   Prothero-Robinson u' = -sigma (u - cos t) - sin t, split
                      f1 = -sigma (u - cos t) (stiff), f2 = -sin t — the
                      reference's own mode-2 problem (mrsdc_test.cpp:23-35,
                      acceptance_test.cpp:357-371), one component per block
  robertson(ncell)    ncell independent Robertson-type kinetics cells (3
                      species, rates scaled per cell): f1 block-local with
                      block 3 (contiguous or interleaved layout); f2 a weak
                      cross-cell exchange of species 0 plus a time forcing
"""
import math

import numpy as np

K1, K2, K3 = 0.4, 30.0, 3.0e3


def _idx(ncell, inter):
    """index[c, j] of component j of cell c."""
    c = np.arange(ncell)[:, None]
    j = np.arange(3)[None, :]
    return j * ncell + c if inter else c * 3 + j


def robertson_f1(u, ncell, inter, xp=np):
    idx = _idx(ncell, inter)
    y = [u[idx[:, j]] for j in range(3)]
    s = 1.0 + 0.25 * xp.arange(ncell, dtype=xp.float64) if xp is np else \
        1.0 + 0.25 * xp.arange(ncell, dtype=xp.float64, device=u.device)
    r1 = (K1 * s) * y[0]
    r2 = (K2 * s) * (y[1] * y[2])
    r3 = (K3 * s) * (y[1] * y[1])
    out = xp.zeros_like(u)
    out[idx[:, 0]] = r2 - r1
    out[idx[:, 1]] = (r1 - r2) - r3
    out[idx[:, 2]] = r3
    return out


def robertson_f2(t, u, ncell, inter, xp=np):
    idx = _idx(ncell, inter)
    y0 = u[idx[:, 0]]
    nxt = u[idx[(np.arange(ncell) + 1) % ncell, 0]]
    out = xp.zeros_like(u)
    out[idx[:, 0]] = 0.1 * (nxt - y0) + 0.01 * math.sin(t)
    return out


def robertson_u0(ncell, inter):
    u = np.zeros(3 * ncell)
    idx = _idx(ncell, inter)
    u[idx[:, 0]] = 1.0 - 0.05 * np.arange(ncell)
    u[idx[:, 1]] = 1e-3
    u[idx[:, 2]] = 0.02 * np.arange(ncell)
    return u


def oscillator_f1(t, u, sigma):
    return -sigma * (u - math.cos(t))


def oscillator_f2(t, u):
    return u * 0.0 - math.sin(t)


# ---- numpy callbacks for the oracle / reference (ctypes RHS_CB signature)
def np_callbacks(name, **kw):
    """(f1, f2) as python functions f(t, u_ptr, out_ptr, n, ctx)."""
    def wrap(fn):
        def cb(t, up, op, n, ctx):
            u = np.ctypeslib.as_array(up, shape=(n,))
            out = np.ctypeslib.as_array(op, shape=(n,))
            out[:] = fn(t, u.copy())
        return cb
    if name == "oscillator":
        sigma = kw["sigma"]
        return wrap(lambda t, u: oscillator_f1(t, u, sigma)), wrap(oscillator_f2)
    if name == "robertson":
        nc, inter = kw["ncell"], kw["inter"]
        return (wrap(lambda t, u: robertson_f1(u, nc, inter)),
                wrap(lambda t, u: robertson_f2(t, u, nc, inter)))
    if name == "quadratic":  # mrsdc_test.cpp:215-228: w = c + beta w^2 has no root
        return wrap(lambda t, u: u * u), wrap(lambda t, u: u * 0.0)
    raise KeyError(name)
