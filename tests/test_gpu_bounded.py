"""GPU parity of the non-periodic boundary closure (bounded.cu through the C
ABI smc_apply_narrow_bounded / smc_first_derivative_bounded) against the
oracle (or_apply_narrow_bounded / or_first_derivative_bounded, pinned in
tests/test_oracle_bounded.py).  Tolerance 1e-12 of the line's max (the
kernel fuses multiply-adds; the oracle does not)."""
import numpy as np
import pytest

import paper_1309_7327_b200 as P
from oracle import oracle as O
from conftest import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-12
SMC = (P.SMC_M47, P.SMC_M48)


def _lines(nl, n, seed):
    rng = np.random.default_rng(seed)
    a = 1.0 + 0.4 * rng.random((nl, n))
    u = rng.standard_normal((nl, n))
    return a, u


@pytest.mark.parametrize("n", [8, 9, 16, 33, 256])
def test_narrow_bounded_vs_oracle(cuda, n):
    import torch
    a, u = _lines(37, n, n)
    h = 1.0 / (n - 1)
    ref = np.stack([O.apply_narrow_bounded(SMC, a[l], u[l], h) for l in range(a.shape[0])])
    got = P.apply_narrow_bounded(a, u, h)
    assert rel_err(got, ref) <= TOL
    # device buffers, and a non-default parameter set with its own m36
    m36 = 0.07
    ref2 = np.stack([O.apply_narrow_bounded((0.08, -0.02), a[l], u[l], h, m36=m36)
                     for l in range(a.shape[0])])
    ad, ud = torch.from_numpy(a).to(cuda), torch.from_numpy(u).to(cuda)
    got2 = P.apply_narrow_bounded(ad, ud, h, params=(0.08, -0.02, m36))
    torch.cuda.synchronize()
    assert rel_err(got2.cpu().numpy(), ref2) <= TOL


@pytest.mark.parametrize("n", [8, 12, 64, 1000])
def test_derivative_bounded_vs_oracle(cuda, n):
    a, u = _lines(5, n, 100 + n)
    h = 0.37 / n
    ref = np.stack([O.first_derivative_bounded(u[l], h) for l in range(u.shape[0])])
    got = P.first_derivative_bounded(u, h)
    assert rel_err(got, ref) <= TOL
    one = P.first_derivative_bounded(u[2].copy(), h)
    assert rel_err(one, ref[2]) <= TOL


def test_bounded_convergence_on_device():
    """The GPU closure keeps the stated orders (boundary cell 2nd order for
    diffusion, 3rd for the derivative; interior 8th)."""
    errs = []
    for n in (33, 65):
        x = np.linspace(0.0, 1.0, n)
        h = x[1] - x[0]
        a = 1.0 + 0.5 * np.sin(2.0 * x)
        u = np.exp(np.sin(3.0 * x))
        up = 3.0 * np.cos(3.0 * x) * u
        ex = np.cos(2.0 * x) * up + a * u * (9.0 * np.cos(3.0 * x) ** 2 - 9.0 * np.sin(3.0 * x))
        e = np.abs(P.apply_narrow_bounded(a, u, h) - ex)
        d = np.abs(P.first_derivative_bounded(u, h) - up)
        errs.append((e[0], e[8:-8].max(), d[0], d[8:-8].max()))
    r = np.log2(np.array(errs[0]) / np.array(errs[1]))
    assert r[0] > 1.5 and r[1] > 7.0 and r[2] > 2.5 and r[3] > 7.0, r


def test_bounded_bad_args():
    with pytest.raises(P.SmcInvalidArgument):
        P.apply_narrow_bounded(np.ones(7), np.ones(7), 0.1)
    with pytest.raises(P.SmcInvalidArgument):
        P.apply_narrow_bounded(np.ones(9), np.ones(10), 0.1)
    with pytest.raises(P.SmcInvalidArgument):
        P.first_derivative_bounded(np.ones(16), -1.0)
    with pytest.raises(P.SmcInvalidArgument):
        P.apply_narrow_bounded(np.ones(16), np.ones(16), 0.1, params=(0.1,))
