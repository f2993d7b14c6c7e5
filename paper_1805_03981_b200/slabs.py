"""Multi-GPU x-slab partition with ghost-face halo exchange.

The reference has no parallel path (SPEC.md:17 puts the paper's MPI out of
scope); the paper distributes elements with deal.II/MPI and counts the ghost
exchange inside the operator time.  Here:

* the structured mesh is cut into slabs of whole x-layers, one per rank (one
  process per GPU, ``torch.distributed``);
* a rank numbers its two ghost-reading x-layers (first and last) first, as
  one contiguous element range, then its interior with x fastest, as in the
  single-domain numbering (``_local_order``; x-neighbour face nodes are
  scattered across the element tile, so x-neighbours are kept adjacent);
* neighbours across a slab edge become ghost codes ``-2 - g``: slot g < L is
  the left ghost layer, L <= g < 2L the right one (L = elements per layer);
  the kernels read those faces from a (2L, d+1, n^(d-1)) ghost buffer;
* each operator application packs the rank's two exported face layers
  (``wk_pack_halo``), exchanges them with the x-neighbour ranks (NCCL P2P
  over NVLink via ``torch.distributed.batch_isend_irecv``) on a high-priority
  halo stream, and overlaps pack + transfer + boundary launch with the
  interior launch on the compute stream (``SlabOperator.apply``).  There is
  no other collective in the time loop.

The per-element arithmetic does not depend on the ordering or on where a
neighbour's face values come from, so the P-rank result is bitwise equal to
the one-GPU result (tests/test_slabs.py, tests/test_gpu_slabs.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import rules
from .mesh import Mesh, Material, AffineGeometry

SLAB_ORDER = "xfast"   # local element numbering of a slab (_local_order)


@dataclass
class SlabPartition:
    """Element bookkeeping of one rank's slab."""
    rank: int
    nranks: int
    d: int
    n_per_dim: tuple
    x0: int
    x1: int
    global_ids: np.ndarray        # (E_local,) global element of each local element
    neighbors: np.ndarray         # (E_local, d, 2) local ids / -1 wall / -2-g ghost
    layer: int                    # L, elements per x-layer
    left_peer: int | None         # rank owning the left ghost layer
    right_peer: int | None
    export_elem: np.ndarray       # local elements whose faces are packed
    export_face: np.ndarray       # face index 2m+s of each export entry
    n_left_export: int
    order: str = "xslow"          # local numbering (_local_order)

    @property
    def n_local(self) -> int:
        return self.global_ids.size

    @property
    def n_ghost(self) -> int:
        return 2 * self.layer if self.nranks > 1 else 0

    def boundary_ranges(self):
        """Local element ranges that read ghost faces: first / last layer."""
        L, E = self.layer, self.n_local
        if self.nranks == 1:
            return []
        if self.x1 - self.x0 <= 2:
            return [(0, E)]
        if self.order == "xfast":
            return [(0, 2 * L)]
        return [(0, L), (E - L, L)]

    def interior_range(self):
        L, E = self.layer, self.n_local
        if self.nranks == 1:
            return (0, E)
        if self.x1 - self.x0 <= 2:
            return (0, 0)
        if self.order == "xfast":
            return (2 * L, E - 2 * L)
        return (L, E - 2 * L)


def slab_bounds(n0: int, nranks: int):
    """Contiguous x-ranges, sizes differing by at most one layer."""
    if nranks > n0:
        raise ValueError(f"cannot cut {n0} x-layers into {nranks} slabs")
    base, extra = divmod(n0, nranks)
    bounds, x = [], 0
    for r in range(nranks):
        w = base + (1 if r < extra else 0)
        bounds.append((x, x + w))
        x += w
    return bounds


def _local_order(nx: int, L: int, nranks: int, order: str):
    """(x-layer-local index ``lay``, slab x index ``xi``) of every local id.

    ``"xslow"``: local id = lay + L xi (x slowest; the first and last layers
    are the two ends of the range).  ``"xfast"``: with one rank the global
    numbering itself (x fastest); with several, the two ghost-reading layers
    first ([xi = 0 | xi = nx-1], each in ``lay`` order), then the interior with
    x fastest, so x-neighbours (whose face nodes are scattered across the
    element tile) stay adjacent in memory as in the single-domain numbering.
    """
    if order not in ("xslow", "xfast"):
        raise ValueError(f"unknown slab order {order!r}")
    lidx = np.arange(nx * L)
    if order == "xslow" or (nranks > 1 and nx <= 2):
        return lidx % L, lidx // L
    if nranks == 1:
        return lidx // nx, lidx % nx
    lay = np.empty_like(lidx)
    xi = np.empty_like(lidx)
    lay[:L], xi[:L] = lidx[:L], 0
    lay[L:2 * L], xi[L:2 * L] = lidx[:L], nx - 1
    t = lidx[2 * L:] - 2 * L
    lay[2 * L:], xi[2 * L:] = t // (nx - 2), 1 + t % (nx - 2)
    return lay, xi


def partition(mesh: Mesh, rank: int, nranks: int, order: str | None = None) -> SlabPartition:
    """Slab of ``rank`` for a structured mesh (build_cartesian numbering);
    ``order`` = local element numbering (``_local_order``, default
    ``SLAB_ORDER``)."""
    d = mesh.d
    nn = tuple(int(v) for v in mesh.n_per_dim)
    n0 = nn[0]
    x0, x1 = slab_bounds(n0, nranks)[rank]
    nx = x1 - x0
    rest = int(np.prod(nn[1:]))          # L: elements per x-layer
    lidx = np.arange(nx * rest)
    lay, xi = _local_order(nx, rest, nranks, SLAB_ORDER if order is None else order)
    i0 = x0 + xi
    gid = i0 + n0 * lay                  # global id = i0 + n0 (i1 + n1 i2)
    # global -> local map for this slab
    g2l = -np.ones(mesh.n_elements, dtype=np.int64)
    g2l[gid] = lidx
    gn = mesh.neighbors[gid]             # (E, d, 2) global neighbour ids
    nbr = np.where(gn >= 0, g2l[np.maximum(gn, 0)], -1).astype(np.int64)
    periodic = mesh.boundary_kind == "periodic"
    left_peer = right_peer = None
    if nranks > 1:
        left_peer = (rank - 1) % nranks if (periodic or rank > 0) else None
        right_peer = (rank + 1) % nranks if (periodic or rank < nranks - 1) else None
        # neighbours outside the slab -> ghost codes
        outside = (gn >= 0) & (nbr < 0)
        # only x-faces can leave the slab
        assert not outside[:, 1:].any()
        first = xi == 0
        last = xi == nx - 1
        left_ghost = outside[:, 0, 0]
        right_ghost = outside[:, 0, 1]
        nbr[left_ghost, 0, 0] = -2 - lay[left_ghost]
        nbr[right_ghost, 0, 1] = -2 - (rest + lay[right_ghost])
        assert np.all(first[left_ghost]) and np.all(last[right_ghost])
    exp_e, exp_f = [], []
    n_left = 0
    if left_peer is not None:
        exp_e.append(lidx[xi == 0])
        exp_f.append(np.zeros(rest, dtype=np.int32))          # face (0, 0)
        n_left = rest
    if right_peer is not None:
        exp_e.append(lidx[xi == nx - 1])
        exp_f.append(np.ones(rest, dtype=np.int32))           # face (0, 1)
    export_elem = np.concatenate(exp_e) if exp_e else np.zeros(0, dtype=np.int64)
    export_face = np.concatenate(exp_f).astype(np.int32) if exp_f else np.zeros(0, np.int32)
    return SlabPartition(rank, nranks, d, nn, x0, x1, gid, nbr, rest, left_peer, right_peer,
                         export_elem.astype(np.int64), export_face, n_left,
                         SLAB_ORDER if order is None else order)


def local_mesh(mesh: Mesh, part: SlabPartition) -> Mesh:
    """Local mesh view (element / vertex arrays restricted, ghost neighbour codes)."""
    return Mesh(mesh.d, mesh.n_per_dim, mesh.vertices, mesh.elements[part.global_ids],
                part.neighbors, mesh.boundary_kind)


def local_material(material: Material, part: SlabPartition) -> Material:
    return Material(c=np.asarray(material.c)[part.global_ids],
                    rho=np.asarray(material.rho)[part.global_ids])


def local_geometry(geo: AffineGeometry, part: SlabPartition) -> AffineGeometry:
    g = part.global_ids
    return AffineGeometry(geo.degree, geo.G[g], geo.det[g], geo.normal[g], geo.fscale[g],
                          geo.h_min, np.asarray(geo.cartesian_flag)[g])


def scatter_state(u_global: np.ndarray, part: SlabPartition) -> np.ndarray:
    return np.ascontiguousarray(u_global[part.global_ids])


def gather_into(u_global: np.ndarray, u_local: np.ndarray, part: SlabPartition) -> None:
    u_global[part.global_ids] = u_local


# ---------------------------------------------------------------------------
# halo exchange


def exchange(send, ghost, part: SlabPartition, dist=None):
    """Post the halo exchange; returns the request list (call .wait()).

    ``send`` = [left export | right export] (packed face layers), ``ghost`` =
    [left ghost layer | right ghost layer].  Rightward traffic is posted before
    leftward traffic on every rank, so with two ranks (left peer == right
    peer) the two messages of a pair still match in order.
    """
    if dist is None:
        import torch.distributed as dist
    L = part.layer
    ops = []
    nl = part.n_left_export
    if part.right_peer is not None:
        ops.append(dist.P2POp(dist.isend, send[nl:nl + L], part.right_peer, tag=0))
    if part.left_peer is not None:
        ops.append(dist.P2POp(dist.irecv, ghost[:L], part.left_peer, tag=0))
    if part.left_peer is not None:
        ops.append(dist.P2POp(dist.isend, send[:L], part.left_peer, tag=1))
    if part.right_peer is not None:
        ops.append(dist.P2POp(dist.irecv, ghost[L:], part.right_peer, tag=1))
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


class SlabOperator:
    """One rank's operator + halo machinery (GPU).

    ``exchange_fn(send, ghost)`` posts the transfer and returns objects with
    ``wait()``; by default the torch.distributed exchange above.  Tests pass a
    loopback that copies between slab operators of one process.
    """

    def __init__(self, mesh: Mesh, geometry: AffineGeometry, material: Material,
                 part: SlabPartition, device="cuda", exchange_fn=None, overlap=True):
        import torch
        from .operator import AcousticOperator
        from ._lib import check, lib
        self.part = part
        self.op = AcousticOperator(local_mesh(mesh, part), local_geometry(geometry, part),
                                   local_material(material, part), device=device,
                                   n_ghost_faces=part.n_ghost)
        self.torch = torch
        C, NF = mesh.d + 1, (geometry.degree + 1) ** (mesh.d - 1)
        self.ghost = torch.zeros((max(part.n_ghost, 1), C, NF), dtype=torch.float64,
                                 device=self.op.device)
        self.send = torch.zeros((max(part.export_elem.size, 1), C, NF), dtype=torch.float64,
                                device=self.op.device)
        if part.n_ghost:
            check(lib().wk_set_ghost_buffer(self.op._ctx, self.op._ptr(self.ghost)))
            ee = np.ascontiguousarray(part.export_elem, dtype=np.int64)
            ef = np.ascontiguousarray(part.export_face, dtype=np.int32)
            from ._lib import dptr
            check(lib().wk_set_halo_exports(self.op._ctx, ee.size, dptr(ee), dptr(ef)))
        self.exchange_fn = exchange_fn or (lambda s, g: exchange(s, g, part))
        self.overlap = overlap
        self._lib, self._check = lib, check
        self._halo = None

    def _range(self, begin, count):
        self._check(self._lib().wk_set_element_range(self.op._ctx, int(begin), int(count)))

    def pack(self, u):
        if self.part.n_ghost:
            self._check(self._lib().wk_pack_halo(self.op._ctx, self.op._ptr(u),
                                                 self.op._ptr(self.send), self.op.stream))

    def apply(self, u, launch):
        """Run ``launch()`` (one fused operator kernel) over the slab with the
        halo exchange of ``u`` overlapped with the interior elements.

        Schedule (overlap): the halo stream (high priority) waits for the
        compute stream, packs the export faces, posts the exchange, waits for
        it and launches the boundary range; the interior range is launched on
        the compute stream after those host calls, so the pack's blocks are
        placed first and the boundary kernel fills the SMs as the interior's
        persistent CTAs retire.  The two concurrent launches use different
        tile-queue counters (``wk_set_queue_slot``); the compute stream then
        waits for the halo stream."""
        if not self.part.n_ghost:
            self._range(0, -1)
            launch()
            return
        if not self.overlap:
            self.pack(u)
            for r in self.exchange_fn(self.send, self.ghost):
                r.wait()
            self._range(0, -1)
            launch()
            return
        torch = self.torch
        main = torch.cuda.current_stream(self.op.device)
        halo = self._halo_stream()
        halo.wait_stream(main)
        with torch.cuda.stream(halo):
            self.pack(u)
            for r in self.exchange_fn(self.send, self.ghost):
                r.wait()
            self._slot(1)
            for b, n in self.part.boundary_ranges():
                self._range(b, n)
                launch()
        self._slot(0)
        b, n = self.part.interior_range()
        if n > 0:
            self._range(b, n)
            launch()
        main.wait_stream(halo)
        self._range(0, -1)

    def _halo_stream(self):
        if self._halo is None:
            self._halo = self.torch.cuda.Stream(self.op.device, priority=-1)
        return self._halo

    def _slot(self, slot):
        self._check(self._lib().wk_set_queue_slot(self.op._ctx, int(slot)))

    def launch_all(self, launch):
        """Launch over the whole slab (ghost buffer already filled)."""
        self._range(0, -1)
        launch()

    def lsrk_stage(self, u_in, u_out, r, a, b, dt, r_dead=False):
        op = self.op
        self.apply(u_in, lambda: self._check(self._lib().wk_lsrk_stage_ex(
            op._ctx, op._ptr(u_in), op._ptr(u_out), op._ptr(r), float(a), float(b),
            float(dt), int(r_dead), op.stream)))

    def ader_step(self, U, V, Y, dt, variant="ader_hdg", reduction="every_second"):
        """One ADER step: halo of U before kernel A (HDG only), halo of Y
        before kernel B; U is updated in place."""
        from . import _lib
        op, lib = self.op, self._lib
        var = _lib.WK_ADER_HDG if variant == "ader_hdg" else _lib.WK_ADER
        pol = _lib.POLICY[reduction]
        launch_a = lambda: self._check(lib().wk_ader_a(
            op._ctx, var, pol, op._ptr(U), op._ptr(V), op._ptr(Y), float(dt), op.stream))
        if var == _lib.WK_ADER_HDG:
            self.apply(U, launch_a)
        else:
            self.launch_all(launch_a)
        self.apply(Y, lambda: self._check(lib().wk_ader_b(
            op._ctx, var, op._ptr(U), op._ptr(V), op._ptr(Y), op.stream)))

    def lsrk_step(self, u, u2, r, dt, scheme):
        """One LSRK step; returns the tensor holding the new state."""
        cur, nxt = u, u2
        for i, (a, b) in enumerate(zip(scheme.a, scheme.b)):
            self.lsrk_stage(cur, nxt, r, a, b, dt, r_dead=(i == scheme.stages - 1))
            cur, nxt = nxt, cur
        return cur


# ---------------------------------------------------------------------------
# bench entry for torchrun (N > 1)


def bench_main(args, rank, world, local, metric, clock_sampler=None, hbm_peak=None,
               hbm_src=None, config=None):
    """The bench under torchrun (one rank per GPU).

    ``--config c5`` (the default): BASELINE config 5 itself, the 128x128x64
    k=4 mesh cut into ``world`` x-slabs -- STRONG scaling, LSRK45 (``value``)
    and ADER-HDG order 5 (``ader_hdg``).  Any other config: weak scaling, a
    32^3 config-2 slab per GPU of a (32 N) x 32 x 32 mesh.  The halo exchange
    runs every operator application (LSRK45: 5 per step, ADER-HDG: 2).  K
    steps timed with CUDA events on every rank, ``args.repeats`` times, the
    median of the per-repeat MAX over ranks (all_reduce MAX); rank 0 prints
    the JSON line.  Also: the end-to-end number (pinned host slab in, K
    steps, slab out, max over ranks) and the SM clocks during the timed
    region (``clock_sampler``)."""
    import contextlib
    import json
    import statistics
    import torch
    import torch.distributed as dist
    from . import configs
    from . import mesh as M
    from .stepping import LSRK45, compute_dt

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    k = 4
    strong = getattr(args, "config", "c5") == "c5"
    if strong:
        # BASELINE config 5: per-cell rho, c ~ U(0.5, 2) from seed 7, Fourier p seed 5
        dims = (128, 128, 64)
        mesh = M.build_cartesian(dims, 3, "periodic")
        mat = configs.random_material(mesh.n_elements, seed=7)
        seed = 5
    else:
        n = 32
        dims = (n * world, n, n)
        mesh = M.build_cartesian(dims, 3, "periodic")
        mat = M.Material.uniform(mesh)
        seed = 2
        config = {"workload": f"c2 per GPU: ({n * world})x{n}x{n} periodic k=4 LSRK45, "
                              "x-slabs (weak scaling)", "scheme": "lsrk45",
                  "parallelism": f"{world} x-slabs (one per GPU)"}
    geo = M.affine_geometry(mesh, k)
    part = partition(mesh, rank, world)
    sub = M.Mesh(3, mesh.n_per_dim, mesh.vertices, mesh.elements[part.global_ids],
                 mesh.neighbors[part.global_ids], mesh.boundary_kind)
    x = M.map_points(sub, rules.gl_points(k))
    p = configs.fourier_pressure(x, seed=seed)
    del x
    u0 = np.zeros((part.n_local, 4) + (k + 1,) * 3)
    u0[:, 3] = p
    del p
    sop = SlabOperator(mesh, geo, mat, part)
    dt = compute_dt(0.2, mesh, mat, k)
    cur = torch.from_numpy(u0).cuda()
    nxt, r = torch.empty_like(cur), torch.empty_like(cur)

    def steps(cur, nxt, count):
        for _ in range(count):
            res = sop.lsrk_step(cur, nxt, r, dt, LSRK45)
            if res is nxt:
                cur, nxt = nxt, cur
        return cur, nxt

    def max_over_ranks(v):
        t = torch.tensor([float(v)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    repeats = max(1, int(getattr(args, "repeats", 3)))
    cur, nxt = steps(cur, nxt, args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    sampler = clock_sampler(local) if (clock_sampler is not None and rank == 0) \
        else contextlib.nullcontext()
    reps = []
    with sampler as clk:
        for _ in range(repeats):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            cur, nxt = steps(cur, nxt, args.steps)
            e1.record()
            torch.cuda.synchronize()
            dist.barrier()
            reps.append(max_over_ranks(e0.elapsed_time(e1)))
    total_ms = statistics.median(reps)
    assert bool(torch.isfinite(cur).all())
    dofs_local = part.n_local * 4 * (k + 1) ** 3
    dofs = int(mesh.n_elements) * 4 * (k + 1) ** 3

    # end to end: pinned host slab in, K steps, slab out (every rank)
    host = torch.from_numpy(u0).pin_memory()
    out_host = torch.empty_like(host).pin_memory()
    torch.cuda.synchronize()
    dist.barrier()
    f0, f1 = torch.cuda.Event(True), torch.cuda.Event(True)
    f0.record()
    cur.copy_(host, non_blocking=True)
    cur, nxt = steps(cur, nxt, args.steps)
    out_host.copy_(cur, non_blocking=True)
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    state_bytes = dofs_local * 8

    # ADER-HDG (order k+1) on the same slabs: 2 halo exchanges per step
    ader = None
    if strong:
        del nxt, r
        U = cur
        V, Y = torch.empty_like(U), torch.empty_like(U)
        U.copy_(host)
        dta = compute_dt(0.1, mesh, mat, k)
        for _ in range(args.warmup):
            sop.ader_step(U, V, Y, dta)
        reps_a = []
        for _ in range(repeats):
            torch.cuda.synchronize()
            dist.barrier()
            g0, g1 = torch.cuda.Event(True), torch.cuda.Event(True)
            g0.record()
            for _ in range(args.steps):
                sop.ader_step(U, V, Y, dta)
            g1.record()
            torch.cuda.synchronize()
            reps_a.append(max_over_ranks(g0.elapsed_time(g1)))
        assert bool(torch.isfinite(U).all())
        ms_a = statistics.median(reps_a) / args.steps
        ader = {"value": dofs / (ms_a * 1e-3), "unit": "DoF/s", "ms_per_step": ms_a,
                "steps": args.steps, "repeats_ms": reps_a,
                "hbm_frac_step_per_gpu": 48.0 * dofs_local / (ms_a * 1e-3) / 1e9 / hbm_peak
                if hbm_peak else None,
                "note": "ADER-HDG order k+1 on the same slabs, 2 halo exchanges per step"}

    if rank == 0:
        # LSRK45: 5 x 32 B/DoF minus the r read of stage 1 and the dead r store of stage 5
        per_gpu_gbs = 144.0 * dofs_local * args.steps / (total_ms * 1e-3) / 1e9
        line = {
            "metric": metric, "value": dofs * args.steps / (total_ms * 1e-3), "unit": "DoF/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "repeats_ms": reps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Fourier-mode pressure, BASELINE rules)",
            "config": config,
            "e2e": {"value": dofs * args.steps / (e2e_ms * 1e-3), "unit": "DoF/s",
                    "h2d_bytes_per_step": state_bytes * world / args.steps,
                    "d2h_bytes_per_step": state_bytes * world / args.steps,
                    "api": "per rank: pinned host slab -> device, K slab LSRK45 steps, "
                           "device -> pinned host (max over ranks)"},
            "gpu_launches": args.steps * 5 * (4 if world > 1 else 1),
            "comm": {"backend": "nccl", "exchanges_per_step": 5 if world > 1 else 0,
                     "bytes_per_exchange_per_rank": 2 * part.layer * 4 * (k + 1) ** 2 * 8
                     if world > 1 else 0,
                     "pattern": "ncclSend/ncclRecv to the x-neighbour ranks (periodic ring), "
                                "overlapped with the interior elements"},
        }
        if hbm_peak:
            line["roofline"] = {
                "bound": "hbm", "achieved": per_gpu_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": per_gpu_gbs / hbm_peak, "traffic": None,
                "kernel": "LSRK45 step per GPU (stage kernels + halo pack, NCCL)",
                "peak_source": hbm_src,
                "algorithmic_bytes": "144 B/DoF per step of the rank's slab (SURVEY 8d's 160 minus "
                                     "the first stage's r read and the last stage's dead r store)"}
        if clock_sampler is not None:
            line["clocks"] = clk.summary()
        if ader is not None:
            line["ader_hdg"] = ader
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
