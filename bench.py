"""Benchmark: FP64 DoF/s per time step of the fused DG-acoustics hot path.

Default workload (N=1): BASELINE config 2 — 3D 32^3 periodic hex mesh, k=4,
LSRK45 (the configuration BASELINE.json's metric is quoted on that fits one
GPU).  A "step" is one full LSRK45 time step (5 fused stage kernels) over the
device-resident state.  The line also carries the ADER-HDG step of the same
mesh, the roofline of the dominant kernel, the CPU baseline (the oracle port
timed on this host's cores on a bounded sample) and the end-to-end number
through the public API with host buffers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c1..c5] [--scheme lsrk45|ader_hdg|...]

With --impl reference the CPU oracle (the reference algorithm restated in
numpy, pinned to the reference's golden vectors) runs on the host cores with
all threads it can use, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 DoF/s per time step (LSRK & ADER) at 1/2/4/8 B200; % of roofline"
BYTES_PER_DOF = {"lsrk45": 160.0, "lsrk59": 288.0, "ader_hdg": 48.0, "ader": 40.0}
STAGE_BYTES = 32.0   # per DoF per LSRK stage launch: read u, r; write u, r
# config 3 (curved, k=5): ADER-HDG 48 B/DoF of vectors + the per-point metric
# per K application (28.0 B/DoF) and the reduced-degree TCK metric (5.3 B/DoF),
# 109.3 B/DoF per step
CURVED_ADER_HDG_BYTES = 109.3


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        with open(path) as f:
            hbm = float(json.load(f)["hbm_gbs"])
            src = "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    fp64 = None
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.jsonl")) as f:
            vals = [json.loads(l) for l in f if l.strip()]
        fp64 = max(v["tflops"] for v in vals if v.get("kind") == "dfma")
    except Exception:
        fp64 = 34.2
    return hbm, src, fp64


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.tmp = None

    def __enter__(self):
        try:
            self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.tmp, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or self.tmp is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.tmp.flush()
        rows = []
        with open(self.tmp.name) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.tmp.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[5 + i].lower() in ("active", "1")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
def run_reference(args, rank):
    """CPU arm: the oracle port of the reference algorithm on host threads."""
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    import oracle
    from oracle import stepping as OS
    from oracle.parallel import ThreadedOracle
    from paper_1805_03981_b200 import configs

    scale = args.ref_scale
    with threadpool_limits(1):
        prob = configs.config(args.config, scale=scale)
        m = prob.mesh
        om = oracle.OracleMesh(m.d, m.n_per_dim, m.vertices, m.elements, m.neighbors,
                               m.boundary_kind)
        if args.config == "c3":
            base = oracle.build_cartesian(m.n_per_dim, 3, "periodic")
            geo = oracle.precompute_geometry(base, prob.k, g=5, mapping=configs.c3_mapping)
        else:
            geo = oracle.precompute_geometry(om, prob.k)
        op = oracle.OracleOperator(om, geo, oracle.OracleMaterial(prob.material.c,
                                                                  prob.material.rho))
        scheme = args.scheme
        cr = prob.schemes.get(scheme, (0.2, 1))[0]
        dt = OS.compute_dt(cr, om, prob.material, prob.k)
        threads = min(os.cpu_count() or 1, 8)
        if scheme.startswith("lsrk"):
            th = ThreadedOracle(op, threads)
            coeffs = OS.LSRK45 if scheme == "lsrk45" else OS.LSRK59
            step = lambda u: th.lsrk_step(u, dt, coeffs)
        else:
            threads = 1
            step = lambda u: OS.ader_step(u, dt, op, scheme)
        u = prob.state
        for _ in range(args.warmup):
            u = step(u)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            u = step(u)
        wall = time.perf_counter() - t0
    value = prob.dofs * args.steps / wall
    sample = (f"{args.config} rules at scale {scale} ({m.n_elements} elements, k={prob.k}, "
              f"{prob.dofs} DoF), {scheme}, {args.steps} steps")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DoF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} {scheme} (CPU sample)", "scheme": scheme},
        "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline_sample(config, scheme, budget_s=20.0):
    """Oracle port timed on this host (rank 0, N=1): bounded sample."""
    from threadpoolctl import threadpool_limits
    import oracle
    from oracle import stepping as OS
    from oracle.parallel import ThreadedOracle
    from paper_1805_03981_b200 import configs
    scale = 0.5 if config in ("c2",) else (0.25 if config in ("c4", "c5") else 0.25)
    with threadpool_limits(1):
        prob = configs.config(config, scale=scale)
        m = prob.mesh
        om = oracle.OracleMesh(m.d, m.n_per_dim, m.vertices, m.elements, m.neighbors,
                               m.boundary_kind)
        geo = oracle.precompute_geometry(om, prob.k)
        op = oracle.OracleOperator(om, geo, oracle.OracleMaterial(prob.material.c,
                                                                  prob.material.rho))
        threads = min(os.cpu_count() or 1, 8)
        th = ThreadedOracle(op, threads)
        u = prob.state
        steps, t0 = 0, time.perf_counter()
        while True:
            u = th.lsrk_step(u, 1e-4, OS.LSRK45)
            steps += 1
            wall = time.perf_counter() - t0
            if wall > budget_s or steps >= 5:
                break
        th.close()
    return {"value": prob.dofs * steps / wall, "unit": "DoF/s", "cores": threads,
            "kind": "port",
            "sample": f"oracle LSRK45, {config} rules at scale {scale} "
                      f"({m.n_elements} elements, {prob.dofs} DoF), {steps} steps, "
                      f"{wall:.1f} s"}


def survey_roofline(k, d, scheme, dofs, ms, bpd, hbm_gbs, fp64_tflops):
    """SURVEY.md §8d's roofline of one time step: t_roof = max(B DoF / BW,
    F DoF / FP64) with B the algorithmic bytes per DoF and F the reference
    cost model's flops per DoF (scheme_cost, kernels.py:235-279 — our
    kernels execute fewer, so frac > 1 on the FP64 side is possible);
    frac = t_roof / t_measured."""
    from paper_1805_03981_b200 import cost
    name = {"rk4": "rk4_classic"}.get(scheme, scheme)
    f = cost.scheme_cost(k, d, name).c_scheme_total / ((d + 1) * (k + 1) ** d)
    t_hbm = bpd * dofs / (hbm_gbs * 1e9) * 1e3
    t_fp = f * dofs / ((fp64_tflops or 34.2) * 1e12) * 1e3
    t_roof = max(t_hbm, t_fp)
    return {"bytes_per_dof": bpd, "model_flop_per_dof": f, "t_hbm_ms": t_hbm, "t_fp64_ms": t_fp,
            "bound": "hbm" if t_hbm >= t_fp else "fp64 (reference model flops)",
            "t_roof_ms": t_roof, "frac": t_roof / ms}


def measure_all_configs(torch, W, configs, hbm=6553.3, fp64=34.2):
    """ms/step and DoF/s of every BASELINE config and scheme on this GPU
    (device-resident state, CUDA-graph replay, CUDA events).  Steps per
    config follow BASELINE.json (c1 10, c3 50, c4/c5 20) except c2 (measured
    by the headline)."""
    plan = [("c1", "lsrk45", 10), ("c3", "ader_hdg", 50), ("c4", "ader_hdg", 20),
            ("c4", "lsrk45", 20), ("c5", "lsrk45", 20), ("c5", "ader_hdg", 20)]
    out = {}
    cache = {}
    for cfg, scheme, steps in plan:
        try:
            t0 = time.perf_counter()
            if cfg not in cache:
                cache.clear()
                torch.cuda.empty_cache()
                # config 3's curved metric is evaluated on the GPU (setup_s)
                prob = configs.config(cfg, geometry="device")
                op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
                cache[cfg] = (prob, op)
            prob, op = cache[cfg]
            setup_s = time.perf_counter() - t0
            cr = prob.schemes[scheme][0]
            dt = W.compute_dt(cr, prob.mesh, prob.material, prob.k)
            st = W.make_stepper(W.SchemeConfig(scheme=scheme, courant=cr), op)
            u = torch.from_numpy(prob.state).cuda()
            st.run(u, dt, 6)                      # warm-up + graph capture
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            res = st.run(u, dt, steps)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            bpd = BYTES_PER_DOF.get(scheme, 0.0)
            if cfg == "c3" and scheme == "ader_hdg":
                bpd = CURVED_ADER_HDG_BYTES
            out[f"{cfg}_{scheme}"] = {
                "ms_per_step": ms, "dofs_per_s": prob.dofs / (ms * 1e-3), "dofs": prob.dofs,
                "steps": steps, "courant": cr, "hbm_algorithmic_gbs": bpd * prob.dofs / ms / 1e6,
                "finite": bool(torch.isfinite(res).all()), "setup_s": setup_s,
                "workload": prob.description,
                "roofline": survey_roofline(prob.k, prob.mesh.d, scheme, prob.dofs, ms, bpd,
                                            hbm, fp64)}
            del u, res, st
        except Exception as exc:                   # reported, not fatal
            out[f"{cfg}_{scheme}"] = {"error": str(exc)[:200]}
    cache.clear()
    torch.cuda.empty_cache()
    return out


def ncu_traffic(kernel_tag):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary_latest.json")
    try:
        with open(path) as f:
            data = json.load(f)
        return data.get(kernel_tag, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scheme", default=None)
    ap.add_argument("--ref-scale", type=float, default=0.5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config table (configs 1-5, both schemes)")
    ap.add_argument("--slab-path", action="store_true",
                    help="run the multi-GPU slab bench even at WORLD_SIZE=1 (path check)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.scheme is None:
        args.scheme = {"c1": "lsrk45", "c2": "lsrk45", "c3": "ader_hdg", "c4": "ader_hdg",
                       "c5": "lsrk45"}[args.config]
    if args.impl == "reference":
        if args.config in ("c4", "c5"):
            args.ref_scale = min(args.ref_scale, 0.25)
        if args.config == "c3":
            args.ref_scale = min(args.ref_scale, 0.25)
        args.steps = min(args.steps, 3)
        args.warmup = min(args.warmup, 1)
        run_reference(args, rank)
        return
    if world > 1 or args.slab_path:
        from paper_1805_03981_b200 import slabs
        if "RANK" not in os.environ:   # --slab-path without torchrun: a one-rank job
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0",
                              MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29533"))
        hbm, hbm_src, _ = peaks()
        slabs.bench_main(args, rank, world, local, METRIC, clock_sampler=ClockSampler,
                         hbm_peak=hbm, hbm_src=hbm_src)
        return
    run_single(args)


def run_single(args):
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import _lib, configs
    from paper_1805_03981_b200._lib import check, lib

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    prob = configs.config(args.config)
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    scheme = args.scheme
    cr = prob.schemes.get(scheme, (0.2, 1))[0]
    dt = W.compute_dt(cr, prob.mesh, prob.material, prob.k)
    dofs = prob.dofs
    state_bytes = dofs * 8
    u0 = torch.from_numpy(prob.state).to(dev)
    stepper = W.make_stepper(W.SchemeConfig(scheme=scheme, courant=cr), op)
    hbm, hbm_src, fp64_peak = peaks()

    # warm-up (eager), then record the CUDA graph of the production path
    u = u0.clone()
    res = stepper.run(u, dt, args.warmup)
    if res is not u:
        u.copy_(res)
    stepper.capture(u, dt)
    torch.cuda.synchronize()

    # timed region: exactly K steps of the production path (the fused kernels,
    # replayed from the CUDA graph), CUDA events on the launching stream
    s = torch.cuda.current_stream()
    sp = op.stream
    b1, b2 = stepper.buffers(u)
    n_launch = args.steps * stepper.launches_per_step()
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.synchronize()
        ev_all0 = torch.cuda.Event(enable_timing=True)
        ev_all1 = torch.cuda.Event(enable_timing=True)
        ev_all0.record(s)
        res = stepper.run(u, dt, args.steps)
        ev_all1.record(s)
        torch.cuda.synchronize()
    total_ms = ev_all0.elapsed_time(ev_all1)
    assert bool(torch.isfinite(res).all())
    ms_step = total_ms / args.steps
    value = dofs * args.steps / (total_ms * 1e-3)

    # roofline of the dominant kernel: the same K steps again, launched one
    # by one with a CUDA event pair around every launch (on the stream the
    # kernels run on), so each launch's duration is measured on the device
    launch_ms, launch_bytes, kern_ms = [], [], {}
    torch.cuda.synchronize()
    if scheme.startswith("lsrk"):
        coeffs = W.LSRK45 if scheme == "lsrk45" else W.LSRK59
        cur, nxt, r = u, b1, b2
        for _ in range(args.steps):
            for a, b in zip(coeffs.a, coeffs.b):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
                check(lib().wk_lsrk_stage(op._ctx, op._ptr(cur), op._ptr(nxt), op._ptr(r),
                                          float(a), float(b), float(dt), sp))
                e1.record(s)
                launch_ms.append((e0, e1))
                # stage 1 (a = 0) does not read r: 24 B/DoF, the others 32
                launch_bytes.append((STAGE_BYTES if a != 0.0 else 24.0) * dofs)
                cur, nxt = nxt, cur
        torch.cuda.synchronize()
        launch_ms = [x.elapsed_time(y) for x, y in launch_ms]
        achieved = sum(launch_bytes) / (sum(launch_ms) * 1e-3) / 1e9
        avg = statistics.mean(launch_ms)
        tag = "affine_op_kernel_lsrk"
        unit_note = ("per LSRK stage launch: 32 B/DoF (read u, r; write u, r), 24 B/DoF on "
                     "stage 1 (a=0, r not read); SURVEY 8d's 160 B/DoF/step")
    else:
        variant = _lib.WK_ADER_HDG if scheme == "ader_hdg" else _lib.WK_ADER
        pol = _lib.POLICY["every_second"]
        evs = []
        for _ in range(args.steps):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(s)
            check(lib().wk_ader_a(op._ctx, variant, pol, op._ptr(u), op._ptr(b1), op._ptr(b2),
                                  float(dt), sp))
            e[1].record(s)
            check(lib().wk_ader_b(op._ctx, variant, op._ptr(u), op._ptr(b1), op._ptr(b2), sp))
            e[2].record(s)
            evs.append(e)
        torch.cuda.synchronize()
        ka = [e[0].elapsed_time(e[1]) for e in evs]
        kb = [e[1].elapsed_time(e[2]) for e in evs]
        kern_ms = {"ader_a_ms": statistics.mean(ka), "ader_b_ms": statistics.mean(kb)}
        launch_ms = [x + y for x, y in zip(ka, kb)]
        avg = statistics.mean(launch_ms)
        achieved = BYTES_PER_DOF[scheme] * dofs / (avg * 1e-3) / 1e9
        tag = "ader_step"
        unit_note = f"{BYTES_PER_DOF[scheme]:.0f} B/DoF per ADER step (kernels A + B)"
    traffic = ncu_traffic(tag)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "kernel": tag,
            "peak_source": hbm_src, "algorithmic_bytes": unit_note,
            "avg_launch_ms": avg, **kern_ms,
            "timing": "per-launch CUDA events in an instrumented pass of the same K steps "
                      "(the timed region itself replays the CUDA graph)"}

    # end-to-end through the public API: host (pinned) numpy state in, result out
    host = torch.from_numpy(prob.state.copy()).pin_memory()
    st = W.StateVector(host.numpy(), prob.k, prob.mesh.d)
    W.advance(st, dt, 3 * stepper.GRAPH_STEPS, stepper)   # warm-up incl. graph capture
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = W.advance(st, dt, args.steps, stepper)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    assert np.all(np.isfinite(out.data))
    e2e = {"value": dofs * args.steps / e2e_s, "unit": "DoF/s",
           "h2d_bytes_per_step": state_bytes / args.steps,
           "d2h_bytes_per_step": state_bytes / args.steps,
           "api": "paper_1805_03981_b200.advance(StateVector(pinned numpy), dt, K, "
                  "make_stepper(...)): one H2D of the state, K steps, one D2H"}

    extras = {}
    if not args.no_extras and scheme.startswith("lsrk"):
        # ADER-HDG (order k+1) step on the same mesh: second half of the metric
        st2 = W.make_stepper(W.SchemeConfig(scheme="ader_hdg"), op)
        dta = W.compute_dt(0.1, prob.mesh, prob.material, prob.k)
        ua = u0.clone()
        st2.run(ua, dta, 3)
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        na = max(10, args.steps // 2)
        ea.record(s)
        st2.run(ua, dta, na)
        eb.record(s)
        torch.cuda.synchronize()
        ms_a = ea.elapsed_time(eb) / na
        extras["ader_hdg"] = {
            "value": dofs / (ms_a * 1e-3), "unit": "DoF/s", "ms_per_step": ms_a,
            "steps": na, "roofline_hbm_frac": 48.0 * dofs / (ms_a * 1e-3) / 1e9 / hbm,
            "roofline": survey_roofline(prob.k, prob.mesh.d, "ader_hdg", dofs, ms_a, 48.0, hbm,
                                        fp64_peak),
            "note": "ADER-HDG order k+1, every_second reduction, same mesh/state"}

    if not args.no_extras and not args.no_configs:
        extras["configs"] = measure_all_configs(torch, W, configs, hbm, fp64_peak)

    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(args.config, scheme)
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": "DoF/s", "cores": 0, "kind": "port",
                   "sample": f"failed: {exc}"}

    line = {
        "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded Fourier-mode pressure, BASELINE rules)",
        "config": {"workload": f"{args.config}: {prob.description}", "scheme": scheme,
                   "elements": prob.mesh.n_elements, "degree": prob.k, "dofs": dofs,
                   "courant": cr, "parallelism": "single GPU",
                   "l2": "inputs larger than L2 (3 resident state vectors of "
                         f"{state_bytes / 1e6:.0f} MB each vs 126 MB L2); no flush"},
        "roofline": roof,
        "step_roofline": survey_roofline(prob.k, prob.mesh.d, scheme, dofs, ms_step,
                                         BYTES_PER_DOF.get(scheme, 0.0), hbm, fp64_peak),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": n_launch,
        "clocks": clk.summary(),
        "fp64_peak_tflops": fp64_peak,
    }
    line.update(extras)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
