"""CPU: the NS oracle (oracle/ns_oracle.c) — physics-independent checks, since
no reference implementation pins it (parity unpinned beyond its building
blocks, which test_oracle.py pins bitwise to the reference kernels)."""
import numpy as np

from oracle import oracle as O
from paper_1309_7327_b200 import workloads as W

DX = 1e-4


def _U(n, **kw):
    T, p, uvw, Y = W.ns_primitives(n, **kw)
    return O.ns_conserved(T, p, uvw, Y), T, p


def test_ctoprim_round_trip():
    U, T, p = _U(10)
    T2, p2 = O.ns_temperature_pressure(U)
    assert np.abs(T2 - T).max() <= 1e-9
    assert np.abs(p2 - p).max() <= 1e-9 * p.max()


def test_conservation_and_mass_consistency():
    n = 12
    U, _, _ = _U(n, hot_spot=True)
    r = O.ns_rhs(U, DX, part=1)
    for v in range(4):  # continuity and momentum telescope to zero
        assert abs(r[v].sum()) <= 1e-12 * np.abs(r[v]).max() * r[v].size
    # corrected species fluxes sum to zero: sum_k rhs_k == continuity rhs
    assert np.abs(r[5:].sum(0) - r[0]).max() <= 1e-12 * np.abs(r[0]).max()
    c = O.ns_rhs(U, DX, part=2)
    assert np.abs(c[5:].sum(0)).max() <= 1e-12 * np.abs(c[5:]).max()
    assert np.all(c[:5] == 0.0)
    f = O.ns_rhs(U, DX, part=0)
    assert np.abs(f - (r + c)).max() <= 1e-12 * np.abs(f).max()


def test_uniform_state_is_steady_without_chemistry():
    n = 10
    T = np.full((n, n, n), 1100.0)
    p = np.full((n, n, n), 101325.0)
    uvw = np.zeros((3, n, n, n))
    Y = np.zeros((9, n, n, n))
    Y[0], Y[1], Y[8] = 0.03, 0.22, 0.75
    U = O.ns_conserved(T, p, uvw, Y)
    r = O.ns_rhs(U, DX, part=1)
    assert np.abs(r).max() <= 1e-6 * np.abs(U[4]).max() * 1e-6


def test_spatial_order_of_accuracy():
    """The advection-diffusion RHS of a smooth state converges at ~8th order
    in dx (same physical state on refined grids of one periodic box):
    Richardson on 16/32/64 cells, compared on the coarse nodes."""
    L = 12e-3
    rs = {}
    for n in (16, 32, 64):
        T, p, uvw, Y = W.ns_primitives(n, seed=3)
        rs[n] = O.ns_rhs(O.ns_conserved(T, p, uvw, Y), L / n, part=1)
    for v in (0, 1, 4, 5, 13):
        e1 = np.abs(rs[16][v] - rs[64][v][::4, ::4, ::4]).max()
        e2 = np.abs(rs[32][v][::2, ::2, ::2] - rs[64][v][::4, ::4, ::4]).max()
        assert np.log2(e1 / e2) > 6.5, (v, e1, e2)


def test_threads_do_not_change_bits():
    """The OpenMP loops of the oracle keep each cell's arithmetic, so the RHS
    is bitwise independent of the thread count (as the reference's
    parallel_for, pde_test.cpp:119-133)."""
    U, _, _ = _U(20, hot_spot=True)
    O.set_threads(1)
    r1 = O.ns_rhs(U, DX, part=0)
    O.set_threads(4)
    r4 = O.ns_rhs(U, DX, part=0)
    O.set_threads(0)
    assert np.array_equal(r1, r4)
