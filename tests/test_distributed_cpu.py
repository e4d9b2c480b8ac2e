"""CPU (gloo, world_size 2 and 3): the host logic of the multi-GPU path —
z-slab decomposition, halo message order (also when prev == next at world 2),
multi-field packing — checked against a global periodic box with the oracle.
The GPU kernels' slab mode is checked bitwise against the periodic box in
tests/test_gpu_narrow.py and tests/test_gpu_ns.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1309_7327_b200.distributed import (Slab, exchange_halo, exchange_halo_fields,
                                              allreduce_max)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nzl, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        n = 12
        nzg = nzl * world
        rng = np.random.default_rng(5)
        a = rng.uniform(0.5, 2.0, (nzg, n, n))
        u = rng.standard_normal((nzg, n, n))
        slab = Slab(rank, world, nzl)
        G = slab.ghost
        # local ghosted arrays with garbage in the ghosts
        ua = torch.full((nzl + 2 * G, n, n), np.nan, dtype=torch.float64)
        aa = torch.full((nzl + 2 * G, n, n), np.nan, dtype=torch.float64)
        ua[G:G + nzl] = torch.from_numpy(u[slab.z0:slab.z0 + nzl])
        aa[G:G + nzl] = torch.from_numpy(a[slab.z0:slab.z0 + nzl])
        for r in exchange_halo(ua, slab, dist):
            r.wait()
        for r in exchange_halo(aa, slab, dist):
            r.wait()
        idx = slab.global_planes()
        ok_ghost = np.array_equal(ua.numpy(), u[idx]) and np.array_equal(aa.numpy(), a[idx])
        # the oracle on the ghosted slab equals the global periodic operator on
        # the slab's planes (interior planes only need +-4 planes)
        m, s = O.build_narrow(8, (3557 / 44100, -2083 / 117600))
        loc = O.narrow3d(m, s, aa.numpy().copy(), ua.numpy().copy(), 0.1, 0.1, 0.1)[G:G + nzl]
        glob = O.narrow3d(m, s, a, u, 0.1, 0.1, 0.1)[slab.z0:slab.z0 + nzl]
        ok_op = np.array_equal(loc, glob)
        # multi-field (NS) packing
        F = torch.full((3, nzl + 2 * G, n, n), np.nan, dtype=torch.float64)
        f = np.stack([u, a, u * a])
        F[:, G:G + nzl] = torch.from_numpy(f[:, slab.z0:slab.z0 + nzl])
        exchange_halo_fields(F, slab, dist)
        ok_fields = np.array_equal(F.numpy(), f[:, idx])
        red = allreduce_max(dist)(float(rank))
        q.put((rank, ok_ghost, ok_op, ok_fields, red))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nzl", [(2, 6), (3, 5)])
def test_slab_halo_exchange_gloo(world, nzl):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, nzl, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, ok_ghost, ok_op, ok_fields, red in res:
        assert ok_ghost, f"rank {rank}: ghost planes"
        assert ok_op, f"rank {rank}: slab operator != global operator"
        assert ok_fields, f"rank {rank}: multi-field halo"
        assert red == world - 1


def test_slab_geometry():
    s = Slab(0, 4, 256)
    assert (s.prev, s.next, s.z0, s.nz_global) == (3, 1, 0, 1024)
    assert s.send_up() == (256, 260) and s.recv_down() == (0, 4)
    assert s.send_down() == (4, 8) and s.recv_up() == (260, 264)
    assert s.global_planes()[:4] == [1020, 1021, 1022, 1023]
    assert s.interior_planes() == (4, 252)
