"""Block decomposition of the periodic box into z-slabs, one per GPU, with a
4-plane halo exchanged over NCCL, overlapped with the interior compute
(SURVEY.md §8(e)).

The reacting-NS slab RHS lives in the library (csrc/dist.cu): `Comm` is one
rank of an NCCL communicator (unique id shared over torch.distributed) or of
an in-process group on one device, `NsSlab` this rank's RHS views.  The
exchange runs on the library's communication stream while ctoprim and the
x / y passes work on the interior planes; the kernels read the two halo
blocks in place, so the state is never copied into a ghosted array.  The
torch.distributed classes below (narrow operator slabs, the peer halo, and
DistributedNs, the NS RHS as a device callback with a Python-side exchange)
are the earlier host-orchestrated paths, kept for the narrow operator and as
the gloo-tested statement of the message order the library follows.

Why z-slabs: with 256^3 cells per GPU a slab has 2 halo faces (vs 6 for a 3-D
block), the ghost planes are contiguous in memory (no pack/unpack kernels:
the 4 boundary planes are sent straight from the state array and received
straight into the ghost planes), and x/y stay periodic inside the kernel.
Weak scaling keeps 256^3 per GPU: the global box is nx x ny x (nz * N).

The host logic here (neighbours, plane offsets, message order) is covered on
CPU by tests/test_distributed_cpu.py with the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass

G = 4  # ghost planes (stencil half width S = 4)


@dataclass(frozen=True)
class Slab:
    """Rank `rank` of `world` owns global z planes [z0, z0 + nz)."""
    rank: int
    world: int
    nz: int
    ghost: int = G

    @property
    def z0(self) -> int:
        return self.rank * self.nz

    @property
    def prev(self) -> int:  # neighbour below (periodic)
        return (self.rank - 1) % self.world

    @property
    def next(self) -> int:  # neighbour above (periodic)
        return (self.rank + 1) % self.world

    @property
    def nz_global(self) -> int:
        return self.nz * self.world

    def global_planes(self):
        """Global z index of every plane of the ghosted local array."""
        return [(self.z0 + k - self.ghost) % self.nz_global for k in range(self.nz + 2 * self.ghost)]

    # plane ranges inside the ghosted local array [0, nz + 2G)
    def send_up(self):      # top interior planes -> next rank's bottom ghosts
        return (self.nz, self.nz + self.ghost)

    def recv_down(self):    # bottom ghosts <- prev rank's top interior planes
        return (0, self.ghost)

    def send_down(self):    # bottom interior planes -> prev rank's top ghosts
        return (self.ghost, 2 * self.ghost)

    def recv_up(self):      # top ghosts <- next rank's bottom interior planes
        return (self.nz + self.ghost, self.nz + 2 * self.ghost)

    def interior_planes(self, s: int = 4):
        """Interior planes whose stencil needs no ghost plane."""
        return (s, self.nz - s)


def exchange_ops(u, slab: Slab, dist):
    """P2P ops for one halo exchange of the ghosted array u (planes first).
    Ordered so that, between any pair of ranks (also when prev == next at
    world 2), the k-th send matches the k-th receive: first every rank sends
    up / receives from below, then sends down / receives from above."""
    a, b = slab.send_up()
    c, d = slab.recv_down()
    e, f = slab.send_down()
    g, h = slab.recv_up()
    return [dist.P2POp(dist.isend, u[a:b], slab.next),
            dist.P2POp(dist.irecv, u[c:d], slab.prev),
            dist.P2POp(dist.isend, u[e:f], slab.prev),
            dist.P2POp(dist.irecv, u[g:h], slab.next)]


def exchange_halo(u, slab: Slab, dist) -> list:
    """Start the exchange; returns the requests.  With one rank the ghosts
    are a periodic self-copy."""
    if slab.world == 1:
        a, b = slab.send_up()
        c, d = slab.recv_down()
        e, f = slab.send_down()
        g, h = slab.recv_up()
        u[c:d].copy_(u[a:b])
        u[g:h].copy_(u[e:f])
        return []
    return dist.batch_isend_irecv(exchange_ops(u, slab, dist))


class DistributedNarrow3D:
    """configs[1]/[3]: the narrow operator on this rank's slab of a periodic
    nx x ny x (nz * world) box.  `a_local` holds nz + 2G planes (coefficient
    ghosts filled by the caller or by one exchange at construction)."""

    def __init__(self, a_local, slab: Slab, dx, dy, dz, dist=None, choice=None, exchange_a=True):
        import torch
        from . import Narrow3DSlab
        self.slab, self.dist = slab, dist
        if exchange_a and slab.world > 1:
            for r in exchange_halo(a_local, slab, dist):
                r.wait()
        elif exchange_a:
            exchange_halo(a_local, slab, dist)
        self.op = Narrow3DSlab(a_local, slab.nz, slab.ghost, dx, dy, dz, choice)
        self.op.set_stream(torch.cuda.current_stream())

    def apply(self, u_ghosted, out, overlap: bool = False) -> None:
        """out (nz planes) = operator(u) after refreshing u's ghost planes.

        overlap=False (default): exchange, then one launch over all planes.
        The 4-plane halo is 2 MB per face at 256^2 (a few us over NVLink),
        while splitting the launch into interior + 2 boundary slices costs
        ~40 % of a 0.29 ms step (measured at N=1, the boundary slices are
        short, latency-bound launches), so the split only pays when the
        exchange is slow.  overlap=True: interior planes [4, nz-4) run while
        the exchange is in flight, the boundary planes after it lands."""
        if not overlap:
            for r in exchange_halo(u_ghosted, self.slab, self.dist):
                r.wait()
            self.op.apply_planes(u_ghosted, out, 0, self.slab.nz)
            return
        lo, hi = self.slab.interior_planes()
        reqs = exchange_halo(u_ghosted, self.slab, self.dist)
        self.op.apply_planes(u_ghosted, out, lo, hi)     # needs no ghost
        for r in reqs:
            r.wait()                                     # current stream waits on NCCL
        self.op.apply_planes(u_ghosted, out, 0, lo)
        self.op.apply_planes(u_ghosted, out, hi, self.slab.nz)


# -------------------------------------------------- multi-component (NS)
def exchange_halo_fields(U, slab: Slab, dist) -> None:
    """Halo exchange of a field-major state U[v, plane, y, x] (e.g. the 14
    conserved NS fields): the 4 boundary planes of every field are packed
    into one contiguous message per direction, sent in the order of
    exchange_ops, and unpacked into the ghost planes.  Blocking (the NS
    kernels need every ghost before ctoprim)."""
    a, b = slab.send_up()
    c, d = slab.recv_down()
    e, f = slab.send_down()
    g, h = slab.recv_up()
    if slab.world == 1:
        U[:, c:d].copy_(U[:, a:b])
        U[:, g:h].copy_(U[:, e:f])
        return
    up = U[:, a:b].contiguous()
    down = U[:, e:f].contiguous()
    from_below = up.new_empty(up.shape)
    from_above = down.new_empty(down.shape)
    ops = [dist.P2POp(dist.isend, up, slab.next), dist.P2POp(dist.irecv, from_below, slab.prev),
           dist.P2POp(dist.isend, down, slab.prev), dist.P2POp(dist.irecv, from_above, slab.next)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    U[:, c:d].copy_(from_below)
    U[:, g:h].copy_(from_above)


def allreduce_max(dist, device=None):
    """Reducer for the device steppers' residual (max over ranks, one double
    per sweep, sdc.cpp:20-30 / mrsdc.cpp:23-35).  The NCCL backend reduces
    device tensors only, so the default device is the current CUDA device
    there and the host under gloo."""
    import torch

    def fn(v: float) -> float:
        if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
            return v
        dev = device
        if dev is None:
            dev = (torch.device("cuda", torch.cuda.current_device())
                   if dist.get_backend() == "nccl" else torch.device("cpu"))
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    return fn


class DistributedNs:
    """configs[3]/[4]: the reacting-NS RHS on this rank's z-slab of a periodic
    nx x ny x (nz * world) box; ghosts of the 14 conserved fields are
    exchanged once per RHS and ctoprim/transport are recomputed on them (the
    paper's choice).  .rhs(part) returns an Rhs usable by
    the device steppers (state = the rank's interior cells)."""

    def __init__(self, slab: Slab, nx: int, ny: int, dx: float, dist=None, choice=None):
        import torch
        from . import NsOperator
        self.slab, self.dist = slab, dist
        self.nx, self.ny = nx, ny
        self.ns = NsOperator(nx, ny, slab.nz, dx, choice=choice, zghost=slab.ghost)
        self.U = torch.zeros((14, slab.nz + 2 * slab.ghost, ny, nx), dtype=torch.float64,
                             device="cuda")
        self.dim = 14 * slab.nz * ny * nx

    def apply(self, U_interior, out, part: int = 0) -> None:
        """out = RHS(U) on interior cells (device tensors, 14 x nz x ny x nx)."""
        G, nz = self.slab.ghost, self.slab.nz
        self.U[:, G:G + nz].copy_(U_interior.view(14, nz, self.ny, self.nx))
        if part != 2:  # chemistry is pointwise: no ghosts needed
            exchange_halo_fields(self.U, self.slab, self.dist)
        import torch
        self.ns.set_stream(torch.cuda.current_stream())
        self.ns.rhs_ghosted(self.U, out.view(14, nz, self.ny, self.nx), part)

    def rhs(self, part: int = 0):
        from . import DeviceCallbackRhs
        return DeviceCallbackRhs(self.dim, lambda t, u, out: self.apply(u, out, part))


# ----------------------------------------------- peer halo (no exchange step)
def ipc_export(t) -> bytes:
    """CUDA IPC handle (64 bytes) of a device tensor's allocation base."""
    import ctypes as C
    from . import _capi, check
    buf = C.create_string_buffer(64)
    check(_capi.lib().smc_ipc_export(C.c_void_p(t.data_ptr()), buf))
    return buf.raw


def ipc_import(handle: bytes) -> int:
    """Device pointer (int) of a buffer exported by another process."""
    import ctypes as C
    from . import _capi, check
    p = C.c_void_p()
    check(_capi.lib().smc_ipc_import(handle, C.byref(p)))
    return p.value


class PeerNarrow3D:
    """configs[1]/[3] with the halo read over peer memory: every rank owns two
    interior-only u buffers (double-buffered by step parity) exported by CUDA
    IPC; the slab kernel loads its S ghost planes straight from the
    neighbours' buffers (NVLink peer loads), so there is no exchange step and
    no ghost copy of u.  Per step one stream-ordered one-element all-reduce
    (sync="nccl") orders every rank's writes of buffer (step % 2) before the
    kernels that read it; the other buffer is free for the next step's writes.
    sync="host" (gloo, tests) synchronises the device and uses a host barrier.
    With one rank the neighbours are the rank itself (periodic)."""

    def __init__(self, a_local, slab: Slab, dx, dy, dz, dist=None, choice=None,
                 exchange_a=True, sync: str = "nccl"):
        import torch
        from . import Narrow3DSlab
        self.slab, self.dist, self.sync = slab, dist, sync
        if exchange_a and slab.world > 1:
            for r in exchange_halo(a_local, slab, dist):
                r.wait()
        elif exchange_a:
            exchange_halo(a_local, slab, dist)
        self.op = Narrow3DSlab(a_local, slab.nz, slab.ghost, dx, dy, dz, choice)
        self.op.set_stream(torch.cuda.current_stream())
        import ctypes as C
        from . import _capi, check, device_tensor
        nzg, ny, nx = a_local.shape
        n = slab.nz * ny * nx
        # whole cudaMalloc allocations: an IPC handle maps the allocation base
        self._raw = []
        self.bufs = []
        for _ in range(2):
            p = C.c_void_p()
            check(_capi.lib().smc_device_alloc(8 * n, C.byref(p)))
            self._raw.append(p.value)
            self.bufs.append(device_tensor(p.value, n).view(slab.nz, ny, nx))
            self.bufs[-1].zero_()
        self._imported = []
        if slab.world == 1:
            self.lo = [b.data_ptr() for b in self.bufs]
            self.hi = list(self.lo)
        else:
            mine = [ipc_export(b) for b in self.bufs]
            allh = [None] * slab.world
            dist.all_gather_object(allh, mine)
            cache = {}

            def open_rank(r):
                if r not in cache:
                    cache[r] = [ipc_import(h) for h in allh[r]]
                    self._imported += cache[r]
                return cache[r]
            self.lo = open_rank(slab.prev)
            self.hi = open_rank(slab.next)
        self._tick = torch.zeros(1, dtype=torch.float64, device=a_local.device)

    def buffer(self, step: int):
        """The interior u buffer to fill for this step."""
        return self.bufs[step % 2]

    def apply(self, step: int, out) -> None:
        """out (nz planes) = operator(u of this step) over the peer halo."""
        import torch
        i = step % 2
        if self.slab.world > 1:
            if self.sync == "nccl":
                self.dist.all_reduce(self._tick)        # stream-ordered across GPUs
            else:
                torch.cuda.synchronize()
                self.dist.barrier()
        self.op.apply_peer(self.bufs[i], self.lo[i], self.slab.nz, self.hi[i], out)

    def close(self) -> None:
        """Unmap the neighbours' buffers and free this rank's (after every
        rank's last kernel that reads them)."""
        import ctypes as C
        from . import _capi
        for p in self._imported:
            _capi.lib().smc_ipc_close(C.c_void_p(p))
        self._imported = []
        self.bufs = []
        for p in self._raw:
            _capi.lib().smc_device_free(C.c_void_p(p))
        self._raw = []


# ------------------------------------------------- library slab NS RHS
class Comm:
    """One rank of a z-slab decomposition, owned by the library (smc_comm)."""

    def __init__(self, handle):
        self._h = handle

    @property
    def handle(self):
        return self._h

    @staticmethod
    def nccl(dist=None, device=None) -> "Comm":
        """NCCL communicator over the torch.distributed world (one rank per
        GPU, current device); rank 0 creates the unique id and broadcasts it."""
        import ctypes as C
        from . import _capi, check
        world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
        rank = dist.get_rank() if world > 1 else 0
        uid = [None]
        if rank == 0:
            buf = C.create_string_buffer(128)
            check(_capi.lib().smc_comm_unique_id(buf))
            uid[0] = buf.raw
        if world > 1:
            dist.broadcast_object_list(uid, src=0, device=device)
        h = C.c_void_p()
        check(_capi.lib().smc_comm_init(uid[0], world, rank, C.byref(h)))
        return Comm(h)

    @staticmethod
    def local_group(n: int) -> list:
        """n ranks of one in-process group on the current device."""
        import ctypes as C
        from . import _capi, check
        hs = (C.c_void_p * n)()
        check(_capi.lib().smc_comm_init_local(n, hs))
        return [Comm(C.c_void_p(h)) for h in hs]

    @property
    def rank(self) -> int:
        import ctypes as C
        from . import _capi, check
        r, s = C.c_int(), C.c_int()
        check(_capi.lib().smc_comm_rank(self._h, C.byref(r), C.byref(s)))
        return r.value

    @property
    def size(self) -> int:
        import ctypes as C
        from . import _capi, check
        r, s = C.c_int(), C.c_int()
        check(_capi.lib().smc_comm_rank(self._h, C.byref(r), C.byref(s)))
        return s.value

    def allreduce_max(self, v: float) -> float:
        import ctypes as C
        from . import _capi, check
        d = C.c_double(v)
        check(_capi.lib().smc_comm_allreduce_max(self._h, C.byref(d)))
        return d.value

    def close(self) -> None:
        if self._h:
            from . import _capi
            _capi.lib().smc_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NsSlab:
    """This rank's z-slab (nz planes) of the periodic nx x ny x (nz * size)
    NS box: .full, .advdiff (MRSDC f1), .chem (f2) are Rhs views of dim
    14 nx ny nz over the rank's interior state (device tensors)."""

    def __init__(self, comm: Comm, nx: int, ny: int, nz: int, dx: float, dy=None, dz=None,
                 choice=None):
        import ctypes as C
        from . import _Rhs, StencilChoice, _capi, _params, check
        choice = choice or StencilChoice()
        dy = dy or dx
        dz = dz or dx
        self.comm = comm
        self.shape = (nz, ny, nx)
        hs = [C.c_void_p() for _ in range(3)]
        pp, keep = _params(choice.params)
        check(_capi.lib().smc_ns_slab_create(comm.handle, nx, ny, nz, dx, dy, dz, choice.order,
                                             pp, len(choice.params), C.byref(hs[0]),
                                             C.byref(hs[1]), C.byref(hs[2])))
        self.full, self.advdiff, self.chem = (_Rhs(h) for h in hs)

    def set_stream(self, stream) -> None:
        for r in (self.full, self.advdiff, self.chem):
            r.set_stream(stream)

    def publish(self, u) -> None:
        """In-process groups: the state the neighbours read next (device)."""
        from . import _capi, check, dptr
        check(_capi.lib().smc_ns_slab_publish(self.full.handle, dptr(u)))
