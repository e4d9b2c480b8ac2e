"""GPU parity of the reacting-NS right-hand side (ctoprim, hypterm, narrow
diffterm + transport, wdot) against the CPU oracle oracle/ns_oracle.c on the
configs[0] state generator.  Tolerance (BASELINE.json north_star): per-
component max error <= 1e-10 of the component's max magnitude.  The oracle is
"parity unpinned" beyond its building blocks (no reference NS exists)."""
import numpy as np
import pytest

import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-10
DX = 1e-4


def _state(n, **kw):
    T, p, uvw, Y = W.ns_primitives(n, **kw)
    return O.ns_conserved(T, p, uvw, Y), (T, p, uvw, Y)


def _percomp(a, b):
    return [float(np.abs(a[v] - b[v]).max() / max(np.abs(b[v]).max(), 1e-300))
            for v in range(a.shape[0])]


def test_conserved_from_primitives(cuda):
    U, prims = _state(12)
    Ug = P.ns_conserved(*prims)
    assert max(_percomp(Ug, U)) <= 1e-14


@pytest.mark.parametrize("part", [P.NS_FULL, P.NS_ADVDIFF, P.NS_CHEM])
@pytest.mark.parametrize("n,kw", [(16, {}), (24, {"hot_spot": True}), (32, {}),
                                  (64, {"hot_spot": True})])
def test_ns_rhs_vs_oracle(cuda, part, n, kw):
    """n = 32 is configs[0] (single full RHS, 32^3 periodic, the configs[0]
    state generator); n = 64 runs whole tiles in every direction."""
    U, _ = _state(n, **kw)
    ref = O.ns_rhs(U, DX, part)
    op = P.NsOperator(n, n, n, DX)
    got = (op.full, op.advdiff, op.chem)[part](0.0, U)
    errs = _percomp(got, ref)
    assert max(errs) <= TOL, errs


def test_ns_temperature_pressure(cuda):
    U, (T, p, _, _) = _state(12)
    op = P.NsOperator(12, 12, 12, DX)
    Tg, pg = op.temperature_pressure(U)
    assert np.abs(Tg - T).max() <= 1e-9 and np.abs(pg - p).max() / 1e5 <= 1e-12


def test_ns_split_sums_to_full(cuda):
    U, _ = _state(16)
    op = P.NsOperator(16, 16, 16, DX)
    full = op.full(0.0, U)
    s = op.advdiff(0.0, U) + op.chem(0.0, U)
    assert max(_percomp(s, full)) <= 1e-13


def test_ns_invariants(cuda):
    """Physics-independent checks: continuity/momentum conserve the total
    (telescoping), species RHS sums to the continuity RHS (mass consistency
    of the corrected diffusion fluxes), chemistry conserves mass."""
    n = 16
    U, _ = _state(n, hot_spot=True)
    op = P.NsOperator(n, n, n, DX)
    r = op.advdiff(0.0, U)
    for v in range(4):
        assert abs(r[v].sum()) <= 1e-12 * np.abs(r[v]).max() * r[v].size
    assert np.abs(r[5:].sum(0) - r[0]).max() <= 1e-12 * np.abs(r[0]).max()
    c = op.chem(0.0, U)
    assert np.abs(c[5:].sum(0)).max() <= 1e-12 * np.abs(c[5:]).max()


def test_ns_slab_matches_periodic(cuda):
    """One z-slab with 4 ghost planes (multi-GPU layout) equals the periodic
    box on its planes."""
    import torch
    n, z0, nzl, G = 16, 4, 8, 4
    U, _ = _state(n)
    full = P.NsOperator(n, n, n, DX).full(0.0, U)
    idx = [(z0 + k - G) % n for k in range(nzl + 2 * G)]
    Ug = torch.from_numpy(np.ascontiguousarray(U[:, idx])).to(cuda)
    slab = P.NsOperator(n, n, nzl, DX, zghost=G)
    out = torch.empty((14, nzl, n, n), dtype=torch.float64, device=cuda)
    slab.rhs_ghosted(Ug, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert max(_percomp(got, full[:, z0:z0 + nzl])) <= 1e-13


# anisotropic boxes: whole tiles along x (64) with short y / z extents
@pytest.mark.parametrize("part", [P.NS_FULL, P.NS_ADVDIFF])
@pytest.mark.parametrize("shape,kw", [((16, 16, 64), {}), ((16, 32, 64), {"hot_spot": True}),
                                      # partial y / z tiles of the direction passes, z chunks
                                      # of the fused phase B that do not divide nz
                                      ((52, 40, 32), {"hot_spot": True}), ((40, 24, 96), {})])
def test_ns_rhs_anisotropic_vs_oracle(cuda, part, shape, kw):
    nz, ny, nx = shape
    T, p, uvw, Y = W.ns_primitives(nx, ny=ny, nz=nz, **kw)
    U = O.ns_conserved(T, p, uvw, Y)
    ref = O.ns_rhs(U, DX, part)
    op = P.NsOperator(nx, ny, nz, DX)
    got = (op.full, op.advdiff, op.chem)[part](0.0, U)
    errs = _percomp(got, ref)
    assert max(errs) <= TOL, errs


def test_ns_slab_matches_periodic_anisotropic(cuda):
    """A 16-plane ghosted z-slab of a 64 x 16 x 32 box equals the periodic box."""
    import torch
    nx, ny, n, z0, nzl, G = 64, 16, 32, 8, 16, 4
    T, p, uvw, Y = W.ns_primitives(nx, ny=ny, nz=n)
    U = O.ns_conserved(T, p, uvw, Y)
    full = P.NsOperator(nx, ny, n, DX).full(0.0, U)
    idx = [(z0 + k - G) % n for k in range(nzl + 2 * G)]
    Ug = torch.from_numpy(np.ascontiguousarray(U[:, idx])).to(cuda)
    slab = P.NsOperator(nx, ny, nzl, DX, zghost=G)
    out = torch.empty((14, nzl, ny, nx), dtype=torch.float64, device=cuda)
    slab.rhs_ghosted(Ug, out)
    torch.cuda.synchronize()
    assert max(_percomp(out.cpu().numpy(), full[:, z0:z0 + nzl])) <= 1e-13


def test_ns_rejects_odd_nx(cuda):
    """The direction kernels stage x-contiguous element pairs (16-byte copies),
    so nx must be even; other shape errors as before (std::invalid_argument ->
    SmcInvalidArgument, a ValueError)."""
    with pytest.raises(ValueError, match="nx must be even"):
        P.NsOperator(15, 16, 16, DX)
    with pytest.raises(ValueError):
        P.NsOperator(8, 16, 16, DX)
    P.NsOperator(10, 9, 9, DX)  # smallest even / odd extents that are allowed


@pytest.mark.parametrize("part", [P.NS_FULL, P.NS_ADVDIFF, P.NS_CHEM])
@pytest.mark.parametrize("n", [64, 128])
def test_ns_host_pipeline_matches_device_path(cuda, part, n):
    """Host buffers run the z-chunk pipeline (32-plane chunks reading their
    halo from the neighbouring chunks in place): the same RHS as the device
    path on the periodic box."""
    import torch
    T, p, uvw, Y = W.ns_primitives(n, hot_spot=True)
    U = P.ns_conserved(*(torch.from_numpy(a).to(cuda) for a in (T, p, uvw, Y)))
    op = P.NsOperator(n, n, n, DX)
    f = (op.full, op.advdiff, op.chem)[part]
    dev = f(0.0, U).cpu().numpy()
    Uh = U.cpu().pin_memory()
    host = f(0.0, Uh).numpy()
    errs = [float(np.abs(host[v] - dev[v]).max() / max(np.abs(dev[v]).max(), 1e-300))
            for v in range(14)]
    assert max(errs) <= 1e-13, errs


@pytest.mark.parametrize("part", [P.NS_FULL, P.NS_ADVDIFF])
def test_ns_rhs_unequal_spacings_vs_oracle(cuda, part):
    """dx != dy != dz: every direction pass scales with its own spacing."""
    T, p, uvw, Y = W.ns_primitives(32, ny=24, nz=16, hot_spot=True)
    U = O.ns_conserved(T, p, uvw, Y)
    ref = O.ns_rhs(U, 1e-4, part, dy=2.5e-4, dz=0.6e-4)
    op = P.NsOperator(32, 24, 16, 1e-4, dy=2.5e-4, dz=0.6e-4)
    got = (op.full, op.advdiff)[part](0.0, U)
    assert max(_percomp(got, ref)) <= TOL


def test_ns_host_pipeline_uneven_chunks(cuda):
    """A box whose middle chunks are not a multiple of the chunk size (200
    planes: 27-plane chunks between the 8, 8, 16 ramps)."""
    import torch
    T, p, uvw, Y = W.ns_primitives(32, ny=24, nz=200)
    U = P.ns_conserved(*(torch.from_numpy(a).to(cuda) for a in (T, p, uvw, Y)))
    op = P.NsOperator(32, 24, 200, DX)
    dev = op.full(0.0, U).cpu().numpy()
    host = op.full(0.0, U.cpu().pin_memory()).numpy()
    assert max(_percomp(host, dev)) <= 1e-13


@pytest.mark.parametrize("n,kw", [(16, {}), (48, {"hot_spot": True})])
def test_ns_rhs_sixth_order_vs_oracle(cuda, n, kw):
    """The sixth-order narrow family (half width 3: odd window offsets in the
    direction passes, two-term coefficient-side velocity transform) against
    the oracle with the same stencil."""
    U, _ = _state(n, **kw)
    m36 = P.DEFAULT_M36
    m64, s = O.build_narrow(6, (m36,))
    ref = O.ns_rhs(U, DX, P.NS_FULL, m64=m64, s=s)
    op = P.NsOperator(n, n, n, DX, choice=P.StencilChoice.narrow6(m36))
    got = op.full(0.0, U)
    errs = _percomp(got, ref)
    assert max(errs) <= TOL, errs
    # and the sixth-order operator is not the eighth-order one
    assert max(_percomp(P.NsOperator(n, n, n, DX).full(0.0, U), ref)) > 1e-9
