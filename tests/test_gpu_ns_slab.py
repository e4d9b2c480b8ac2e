"""GPU: the library's z-slab NS RHS (csrc/dist.cu, smc_ns_slab_*) against the
periodic box.

* Several ranks of an in-process group on one device (halo by device copies
  of the neighbours' published states): the slabs' RHS, stacked, equals the
  periodic box's -- the halo blocks, the state view and the interior /
  boundary split of the evaluation.
* One NCCL rank (the whole box; the neighbours are the rank itself, so the
  halo goes through ncclSend / ncclRecv to self): the slab RHS equals the
  periodic box, and the device SDC stepper with the residual reduced over
  the communicator advances it like the periodic operator.
Ranks that wait on each other are never run as separate processes on one GPU
(B200_PROFILING.md); the multi-rank message order is covered on CPU with
gloo (test_distributed_cpu.py)."""
import numpy as np
import pytest

import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W
from paper_1309_7327_b200.distributed import Comm, NsSlab
from oracle import oracle as O

pytestmark = pytest.mark.gpu
DX = 1e-4


def _percomp(a, b):
    """max over components of max |a - b| / max |b| (absolute where b == 0)"""
    return max(float(np.abs(a[v] - b[v]).max() / max(np.abs(b[v]).max(), 1.0 if not
                                                        np.abs(b[v]).max() else 0.0))
               for v in range(a.shape[0]))


@pytest.mark.parametrize("part", [P.NS_FULL, P.NS_ADVDIFF, P.NS_CHEM])
@pytest.mark.parametrize("ranks,nz,shape", [(2, 16, (32, 32)), (3, 16, (64, 32)),
                                            (4, 8, (32, 16))])
def test_local_group_slabs_equal_periodic_box(cuda, part, ranks, nz, shape):
    import torch
    nx, ny = shape
    T, p, uvw, Y = W.ns_primitives(nx, ny=ny, nz=nz * ranks, hot_spot=True)
    U = O.ns_conserved(T, p, uvw, Y)
    ref = (lambda o: (o.full, o.advdiff, o.chem)[part])(P.NsOperator(nx, ny, nz * ranks, DX))(0.0, U)
    comms = Comm.local_group(ranks)
    slabs = [NsSlab(c, nx, ny, nz, DX) for c in comms]
    us = [torch.from_numpy(np.ascontiguousarray(U[:, r * nz:(r + 1) * nz])).to(cuda)
          for r in range(ranks)]
    for s, u in zip(slabs, us):
        s.publish(u)
    outs = []
    for s, u in zip(slabs, us):
        o = torch.empty_like(u)
        (s.full, s.advdiff, s.chem)[part](0.0, u, o)
        outs.append(o)
    torch.cuda.synchronize()
    got = np.concatenate([o.cpu().numpy() for o in outs], axis=1)
    assert _percomp(got, ref) <= 1e-13


def test_nccl_single_rank_slab_equals_periodic_box(cuda):
    import torch
    from paper_1309_7327_b200 import _capi
    n = 32
    T, p, uvw, Y = W.ns_primitives(n, hot_spot=True)
    U = O.ns_conserved(T, p, uvw, Y)
    ref = P.NsOperator(n, n, n, DX).full(0.0, U)
    try:
        comm = Comm.nccl()
    except _capi.SmcError as exc:
        pytest.skip(f"NCCL unavailable: {exc}")
    assert (comm.rank, comm.size) == (0, 1)
    assert comm.allreduce_max(2.5) == 2.5
    slab = NsSlab(comm, n, n, n, DX)
    Ud = torch.from_numpy(U).to(cuda)
    got = slab.full(0.0, Ud)
    torch.cuda.synchronize()
    assert _percomp(got.cpu().numpy(), ref) <= 1e-13


def test_nccl_single_rank_sdc_with_library_reducer(cuda):
    """The device SDC stepper advancing the NCCL slab RHS, residual reduced
    over the communicator in the library: the periodic operator's advance."""
    import torch
    from paper_1309_7327_b200 import _capi
    from test_gpu_ns_steppers import acoustic_dt
    n = 16
    prims = W.ns_primitives(n)
    U = O.ns_conserved(*prims)
    dt = acoustic_dt(prims, DX)
    try:
        comm = Comm.nccl()
    except _capi.SmcError as exc:
        pytest.skip(f"NCCL unavailable: {exc}")
    slab = NsSlab(comm, n, n, n, DX)
    slab.set_stream(torch.cuda.current_stream())
    st = P.SdcStepper(3, P.StepControls(4, 0.0))
    st.set_comm(comm)
    got, d = st.integrate(slab.full, torch.from_numpy(U).to(cuda), 0.0, 2 * dt, 2)
    torch.cuda.synchronize()
    ref, dr = P.SdcStepper(3, P.StepControls(4, 0.0)).integrate(
        P.NsOperator(n, n, n, DX).full, U, 0.0, 2 * dt, 2)
    assert _percomp(got.cpu().numpy(), ref) <= 1e-12
    assert d.fresh_evals == dr.fresh_evals == 2 * 8 + 1


def test_nccl_single_rank_mrsdc_equals_periodic(cuda):
    """MRSDC mode 1 advancing the NCCL slab operators (advection-diffusion
    with the halo exchange, the chemistry part with each fine node's update
    fused into it) equals the periodic operators' advance bit for bit."""
    import torch
    from paper_1309_7327_b200 import _capi
    from test_gpu_ns_steppers import acoustic_dt
    n = 16
    prims = W.ns_primitives(n, ignition=True)
    U = O.ns_conserved(*prims)
    dt = acoustic_dt(prims, DX)
    try:
        comm = Comm.nccl()
    except _capi.SmcError as exc:
        pytest.skip(f"NCCL unavailable: {exc}")
    slab = NsSlab(comm, n, n, n, DX)
    slab.set_stream(torch.cuda.current_stream())
    st = P.MrsdcStepper(3, 5, P.StepControls(3, 0.0))
    st.set_comm(comm)
    got, d = st.integrate_mode1(slab.advdiff, slab.chem, torch.from_numpy(U).to(cuda), 0.0,
                                2 * dt, 2)
    torch.cuda.synchronize()
    op = P.NsOperator(n, n, n, DX)
    ref, dr = P.MrsdcStepper(3, 5, P.StepControls(3, 0.0)).integrate_mode1(
        op.advdiff, op.chem, U, 0.0, 2 * dt, 2)
    assert np.array_equal(got.cpu().numpy(), ref)
    assert d.f2_evals == dr.f2_evals and d.f1_evals == dr.f1_evals


def test_slab_rejects_thin_slabs(cuda):
    comms = Comm.local_group(2)
    with pytest.raises(ValueError):
        NsSlab(comms[0], 32, 32, 2, DX)  # fewer planes than the halo is deep


@pytest.mark.parametrize("part", [P.NS_FULL, P.NS_ADVDIFF, P.NS_CHEM])
def test_nccl_slab_host_pipeline_matches_device_path(cuda, part):
    """Host buffers on an NCCL slab: boundary planes first, the halo
    exchange folded into the chunk pipeline; the same RHS as the device
    path."""
    import torch
    from paper_1309_7327_b200 import _capi
    n = 64
    T, p, uvw, Y = W.ns_primitives(n, hot_spot=True)
    U = O.ns_conserved(T, p, uvw, Y)
    try:
        comm = Comm.nccl()
    except _capi.SmcError as exc:
        pytest.skip(f"NCCL unavailable: {exc}")
    slab = NsSlab(comm, n, n, n, DX)
    f = (slab.full, slab.advdiff, slab.chem)[part]
    dev = f(0.0, torch.from_numpy(U).to(cuda)).cpu().numpy()
    host = f(0.0, torch.from_numpy(U).pin_memory()).numpy()
    assert _percomp(host, dev) <= 1e-13
