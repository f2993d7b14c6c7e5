"""Multi-GPU slabs over REAL NCCL (one process per GPU).

World size 2 (and 4 when present) on the x-slab partition of a periodic
mesh with random materials: LSRK45 and ADER-HDG steps through
``SlabOperator`` (halo stream, pack kernel, ``batch_isend_irecv`` with the
x-neighbour ranks, boundary / interior launches) and the result gathered on
rank 0 must be BITWISE equal to the one-GPU run (element-wise face terms, no
atomics).  Skipped when fewer than two GPUs are visible; the same host logic
is covered with gloo on CPU (tests/test_slabs.py) and the device ghost path
with a one-GPU loopback (tests/test_gpu_slabs.py)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPE, K, STEPS = (16, 8, 6), 4, 3


def _problem():
    from paper_1805_03981_b200 import mesh as M
    mesh = M.build_cartesian(SHAPE, 3, "periodic")
    rng = np.random.default_rng(5)
    mat = M.Material(c=rng.uniform(0.5, 2, mesh.n_elements),
                     rho=rng.uniform(0.5, 2, mesh.n_elements))
    u0 = rng.standard_normal((mesh.n_elements, 4) + (K + 1,) * 3)
    return mesh, M.affine_geometry(mesh, K), mat, u0


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import slabs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    mesh, geo, mat, u0 = _problem()
    part = slabs.partition(mesh, rank, world)
    sop = slabs.SlabOperator(mesh, geo, mat, part)
    dt = W.compute_dt(0.2, mesh, mat, K)
    cur = torch.from_numpy(slabs.scatter_state(u0, part)).cuda()
    nxt, r = torch.empty_like(cur), torch.empty_like(cur)
    for _ in range(STEPS):
        res = sop.lsrk_step(cur, nxt, r, dt, W.LSRK45)
        if res is nxt:
            cur, nxt = nxt, cur
    U = torch.from_numpy(slabs.scatter_state(u0, part)).cuda()
    V, Y = torch.empty_like(U), torch.empty_like(U)
    for _ in range(STEPS):
        sop.ader_step(U, V, Y, 0.5 * dt)
    torch.cuda.synchronize()
    parts = [None] * world if rank == 0 else None
    dist.gather_object((part.global_ids, cur.cpu().numpy(), U.cpu().numpy()), parts, dst=0)
    if rank == 0:
        lsrk = np.empty_like(u0)
        ader = np.empty_like(u0)
        for gids, a, b in parts:
            lsrk[gids] = a
            ader[gids] = b
        np.savez(out_path, lsrk=lsrk, ader=ader)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_slabs_bitwise_equal_one_gpu(world, tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    import paper_1805_03981_b200 as W
    out = str(tmp_path / "slabs.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    mesh, geo, mat, u0 = _problem()
    op = W.AcousticOperator(mesh, geo, mat)
    dt = W.compute_dt(0.2, mesh, mat, K)
    x = torch.from_numpy(u0).cuda()
    ref_l = W.advance(W.StateVector(x, K, 3), dt, STEPS,
                      W.make_stepper(W.SchemeConfig(scheme="lsrk45"), op)).data.cpu().numpy()
    ref_a = W.advance(W.StateVector(x, K, 3), 0.5 * dt, STEPS,
                      W.make_stepper(W.SchemeConfig(scheme="ader_hdg"), op)).data.cpu().numpy()
    assert np.array_equal(got["lsrk"], ref_l)
    assert np.array_equal(got["ader"], ref_a)
