"""Multi-GPU slab logic on CPU: partition bookkeeping and the halo exchange
over torch.distributed (gloo, world sizes 2 and 3)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_03981_b200 import mesh as M
from paper_1805_03981_b200 import slabs

K = 2
C, N = 4, K + 1
NF = N * N


def _face_slice(u, m, s):
    """(E, C, NF) face-node slice of face (m, s), face index order of the kernels."""
    idx = [slice(None)] * 5
    idx[2 + 2 - m] = -1 if s else 0
    return u[tuple(idx)].reshape(u.shape[0], C, NF)


@pytest.mark.parametrize("order", ["xfast", "xslow"])
@pytest.mark.parametrize("nranks", [1, 2, 3, 4])
@pytest.mark.parametrize("bk", ["periodic", "sound_soft"])
def test_partition_bookkeeping(nranks, bk, order):
    mesh = M.build_cartesian((8, 3, 2), 3, bk)
    seen = np.zeros(mesh.n_elements, dtype=int)
    for r in range(nranks):
        p = slabs.partition(mesh, r, nranks, order=order)
        assert p.order == order
        seen[p.global_ids] += 1
        L = p.layer
        for le, g in enumerate(p.global_ids):
            for m in range(3):
                for s in (0, 1):
                    code = p.neighbors[le, m, s]
                    gn = mesh.neighbors[g, m, s]
                    if code >= 0:
                        assert p.global_ids[code] == gn
                    elif code == -1:
                        assert gn == -1
                    else:
                        slot = -2 - code
                        assert m == 0 and gn >= 0
                        # the ghost element lives on the peer rank
                        peer = p.left_peer if slot < L else p.right_peer
                        q = slabs.partition(mesh, peer, nranks, order=order)
                        assert gn in set(q.global_ids.tolist())
        if nranks > 1:
            b = sum(n for _, n in p.boundary_ranges())
            assert b + p.interior_range()[1] == p.n_local
            # the ghost readers are exactly the boundary ranges (periodic:
            # every element of the first / last layer reads one ghost face)
            reads = (p.neighbors <= -2).any(axis=(1, 2))
            in_bnd = np.zeros(p.n_local, dtype=bool)
            for b0, n in p.boundary_ranges():
                in_bnd[b0:b0 + n] = True
            ib, n_int = p.interior_range()
            assert not reads[ib:ib + n_int].any()
            assert np.all(in_bnd[reads])
            assert not in_bnd[ib:ib + n_int].any()
        if nranks == 1 and order == "xfast":
            # one slab = the global numbering itself
            assert np.array_equal(p.global_ids, np.arange(mesh.n_elements))
    assert np.all(seen == 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, nranks, port, bk, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        mesh = M.build_cartesian((6, 3, 2), 3, bk)
        rng = np.random.default_rng(7)
        u = rng.standard_normal((mesh.n_elements, C) + (N,) * 3)
        p = slabs.partition(mesh, rank, nranks)
        ul = u[p.global_ids]
        # pack exactly as wk_pack_halo does: entry i = face export_face[i] of export_elem[i]
        send = np.stack([_face_slice(ul[e:e + 1], f >> 1, f & 1)[0]
                         for e, f in zip(p.export_elem, p.export_face)]) \
            if p.export_elem.size else np.zeros((1, C, NF))
        ghost = torch.zeros((max(p.n_ghost, 1), C, NF), dtype=torch.float64)
        reqs = slabs.exchange(torch.from_numpy(send), ghost, p)
        for r in reqs:
            r.wait()
        # every ghost code must now see the neighbour's opposite face slice
        ok = True
        for le, g in enumerate(p.global_ids):
            for s in (0, 1):
                code = p.neighbors[le, 0, s]
                if code <= -2:
                    gn = mesh.neighbors[g, 0, s]
                    want = _face_slice(u[gn:gn + 1], 0, 1 - s)[0]
                    got = ghost[-2 - code].numpy()
                    ok &= bool(np.array_equal(got, want))
        results[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("bk", ["periodic", "sound_soft"])
def test_halo_exchange_gloo(nranks, bk):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(nranks, _free_port(), bk, results), nprocs=nranks, join=True)
    assert len(results) == nranks and all(results.values())
