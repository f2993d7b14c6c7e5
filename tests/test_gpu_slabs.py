"""Slab decomposition on ONE GPU: P slab operators in one process with a
loopback halo (device copies between their send/ghost buffers).  The
P-slab LSRK45 and ADER-HDG trajectories must be BITWISE equal to the
one-domain run (element-wise faces, no atomics, order-independent
arithmetic), which exercises the ghost-face path of every kernel."""

import numpy as np
import pytest
import torch

import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import mesh as M
from paper_1805_03981_b200 import slabs

pytestmark = pytest.mark.gpu


def _setup(bk, k, shape=(8, 4, 3)):
    mesh = M.build_cartesian(shape, 3, bk)
    geo = M.affine_geometry(mesh, k)
    rng = np.random.default_rng(11)
    mat = M.Material(c=rng.uniform(0.5, 2, mesh.n_elements), rho=rng.uniform(0.5, 2, mesh.n_elements))
    u0 = rng.standard_normal((mesh.n_elements, 4) + (k + 1,) * 3)
    return mesh, geo, mat, u0


def _loopback(sops, us):
    for s, u in zip(sops, us):
        s.pack(u)
    for s in sops:
        p = s.part
        L = p.layer
        if p.left_peer is not None:
            q = sops[p.left_peer]
            s.ghost[:L].copy_(q.send[q.part.n_left_export:q.part.n_left_export + L])
        if p.right_peer is not None:
            q = sops[p.right_peer]
            s.ghost[L:2 * L].copy_(q.send[:L])


@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("bk", ["periodic", "sound_soft"])
def test_slab_lsrk_bitwise(cuda, nranks, bk):
    k = 4
    mesh, geo, mat, u0 = _setup(bk, k)
    op = W.AcousticOperator(mesh, geo, mat)
    dt = 1e-3
    ref = W.advance(W.StateVector(torch.from_numpy(u0).cuda(), k, 3), dt, 2,
                    W.make_stepper(W.SchemeConfig(scheme="lsrk45"), op)).data
    parts = [slabs.partition(mesh, r, nranks) for r in range(nranks)]
    sops = [slabs.SlabOperator(mesh, geo, mat, p) for p in parts]
    cur = [torch.from_numpy(slabs.scatter_state(u0, p)).cuda() for p in parts]
    nxt = [torch.empty_like(c) for c in cur]
    reg = [torch.empty_like(c) for c in cur]
    for _ in range(2):
        for a, b in zip(W.LSRK45.a, W.LSRK45.b):
            _loopback(sops, cur)
            for s, ui, uo, r in zip(sops, cur, nxt, reg):
                s.launch_all(lambda s=s, ui=ui, uo=uo, r=r: s._check(s._lib().wk_lsrk_stage(
                    s.op._ctx, s.op._ptr(ui), s.op._ptr(uo), s.op._ptr(r), float(a), float(b),
                    float(dt), s.op.stream)))
            cur, nxt = nxt, cur
    out = torch.empty_like(ref)
    for p, c in zip(parts, cur):
        out[torch.from_numpy(p.global_ids).cuda()] = c
    assert torch.equal(out, ref)


@pytest.mark.parametrize("nranks", [2, 3])
def test_slab_ader_hdg_bitwise(cuda, nranks):
    k = 3
    mesh, geo, mat, u0 = _setup("periodic", k, (6, 3, 3))
    op = W.AcousticOperator(mesh, geo, mat)
    dt = 1e-3
    ref = W.ader_step(W.StateVector(torch.from_numpy(u0).cuda(), k, 3), dt, op, "ader_hdg").data
    parts = [slabs.partition(mesh, r, nranks) for r in range(nranks)]
    sops = [slabs.SlabOperator(mesh, geo, mat, p) for p in parts]
    U = [torch.from_numpy(slabs.scatter_state(u0, p)).cuda() for p in parts]
    V = [torch.empty_like(x) for x in U]
    Y = [torch.empty_like(x) for x in U]
    from paper_1805_03981_b200 import _lib
    _loopback(sops, U)
    for s, u, v, y in zip(sops, U, V, Y):
        s.launch_all(lambda s=s, u=u, v=v, y=y: s._check(s._lib().wk_ader_a(
            s.op._ctx, _lib.WK_ADER_HDG, _lib.POLICY["every_second"], s.op._ptr(u),
            s.op._ptr(v), s.op._ptr(y), float(dt), s.op.stream)))
    _loopback(sops, Y)
    for s, u, v, y in zip(sops, U, V, Y):
        s.launch_all(lambda s=s, u=u, v=v, y=y: s._check(s._lib().wk_ader_b(
            s.op._ctx, _lib.WK_ADER_HDG, s.op._ptr(u), s.op._ptr(v), s.op._ptr(y),
            s.op.stream)))
    out = torch.empty_like(ref)
    for p, x in zip(parts, U):
        out[torch.from_numpy(p.global_ids).cuda()] = x
    assert torch.equal(out, ref)


def test_slab_overlap_ranges(cuda):
    """Interior/boundary split launches (the overlap schedule) give the same
    result as one launch."""
    k = 4
    mesh, geo, mat, u0 = _setup("periodic", k)
    parts = [slabs.partition(mesh, r, 2) for r in range(2)]
    sops = [slabs.SlabOperator(mesh, geo, mat, p) for p in parts]
    U = [torch.from_numpy(slabs.scatter_state(u0, p)).cuda() for p in parts]
    outs = []
    for split in (False, True):
        res = []
        _loopback(sops, U)
        for s, u in zip(sops, U):
            o = torch.empty_like(u)
            launch = lambda s=s, u=u, o=o: s._check(s._lib().wk_rhs(
                s.op._ctx, s.op._ptr(u), s.op._ptr(o), s.op.stream))
            if split:
                b, n = s.part.interior_range()
                s._range(b, n)
                launch()
                for b, n in s.part.boundary_ranges():
                    s._range(b, n)
                    launch()
                s._range(0, -1)
            else:
                s.launch_all(launch)
            res.append(o)
        outs.append(res)
    for a, b in zip(*outs):
        assert torch.equal(a, b)


class _Done:
    def wait(self):
        pass


@pytest.mark.parametrize("order", ["xfast", "xslow"])
@pytest.mark.parametrize("shape,nranks", [((8, 4, 3), 2), ((8, 4, 3), 3), ((24, 12, 12), 2),
                                          ((64, 32, 16), 4)])
def test_slab_overlap_schedule_bitwise(cuda, order, shape, nranks):
    """The production overlap schedule (SlabOperator.apply: pack, exchange and
    boundary launch on the halo stream with tile-queue slot 1, interior on the
    compute stream with slot 0) for LSRK45 stages and ADER-HDG steps, bitwise
    equal to the one-domain run.  The exchange hook copies the ghost layers a
    loopback pass computed beforehand (on the stream the schedule runs it)."""
    k = 4
    mesh, geo, mat, u0 = _setup("periodic", k, shape)
    op = W.AcousticOperator(mesh, geo, mat)
    dt = 1e-3
    ref = W.advance(W.StateVector(torch.from_numpy(u0).cuda(), k, 3), dt, 2,
                    W.make_stepper(W.SchemeConfig(scheme="lsrk45"), op)).data
    ref_ader = W.ader_step(W.StateVector(ref.clone(), k, 3), dt, op, "ader_hdg").data
    parts = [slabs.partition(mesh, r, nranks, order=order) for r in range(nranks)]
    sops = [slabs.SlabOperator(mesh, geo, mat, p) for p in parts]
    truth = [None] * nranks
    for i, s in enumerate(sops):
        s.exchange_fn = lambda send, ghost, i=i: (ghost.copy_(truth[i]), [_Done()])[1]

    def stage_ghosts(us):
        _loopback(sops, us)
        for i, s in enumerate(sops):
            truth[i] = s.ghost.clone()

    cur = [torch.from_numpy(slabs.scatter_state(u0, p)).cuda() for p in parts]
    nxt = [torch.empty_like(c) for c in cur]
    reg = [torch.empty_like(c) for c in cur]
    for _ in range(2):
        for a, b in zip(W.LSRK45.a, W.LSRK45.b):
            stage_ghosts(cur)
            for s, ui, uo, r in zip(sops, cur, nxt, reg):
                s.lsrk_stage(ui, uo, r, a, b, dt)
            cur, nxt = nxt, cur
    out = torch.empty_like(ref)
    for p, c in zip(parts, cur):
        out[torch.from_numpy(p.global_ids).cuda()] = c
    assert torch.equal(out, ref)
    # ADER-HDG: halo of U before kernel A, of Y before kernel B
    V = [torch.empty_like(c) for c in cur]
    Y = [torch.empty_like(c) for c in cur]
    stage_ghosts(cur)
    from paper_1805_03981_b200 import _lib
    for s, u, v, y in zip(sops, cur, V, Y):
        s.apply(u, lambda s=s, u=u, v=v, y=y: s._check(s._lib().wk_ader_a(
            s.op._ctx, _lib.WK_ADER_HDG, _lib.POLICY["every_second"], s.op._ptr(u),
            s.op._ptr(v), s.op._ptr(y), float(dt), s.op.stream)))
    stage_ghosts(Y)
    for s, u, v, y in zip(sops, cur, V, Y):
        s.apply(y, lambda s=s, u=u, v=v, y=y: s._check(s._lib().wk_ader_b(
            s.op._ctx, _lib.WK_ADER_HDG, s.op._ptr(u), s.op._ptr(v), s.op._ptr(y),
            s.op.stream)))
    for p, c in zip(parts, cur):
        out[torch.from_numpy(p.global_ids).cuda()] = c
    assert torch.equal(out, ref_ader)
