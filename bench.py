"""Benchmark: FP64 DoF/s per time step of the fused DG-acoustics hot path.

Headline workload (every N, N = 1 included): BASELINE config 5 -- the
128x128x64 periodic hex mesh, k = 4 (524 M DoF), per-cell rho, c ~ U(0.5, 2)
(seed 7), seeded Fourier-mode pressure -- advanced by LSRK45 (the metric's
"LSRK" half; ``value``).  The same job's ADER-HDG order-5 step (the "ADER"
half) rides along in ``ader_hdg``.  With N > 1 the mesh is cut into N x-slabs
(strong scaling, one process per GPU, NCCL ghost-face halo overlapped with the
interior elements); ``python bench.py --gpus N`` launches
torchrun itself when it is not already running under it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--repeats R]
                    [--impl b200|reference] [--config c1..c5] [--scheme ...]

A "step" is one full time step (5 fused stage kernels for LSRK45, kernels A +
B for ADER-HDG) over the device-resident state; K steps are timed with CUDA
events on the launching stream, R = 3 times, median reported, max over ranks.

Roofline: LSRK is HBM-bound -- achieved = algorithmic bytes of one stage
launch (32 B/DoF, 24 on stage 1) / its event-timed duration;
``traffic`` = DRAM bytes of one stage launch measured IN THIS RUN by an ncu
subprocess on the same workload (``--probe``).  ADER kernel A is FP64-bound:
its roofline is the EXECUTED FP64 work (ncu: 2 DFMA + DMUL + DADD thread
instructions per launch) over its event-timed duration against the measured
DFMA peak, next to the FP64-pipe utilisation and its HBM fraction.

``--impl reference`` runs the reference algorithm on the host cores: the
oracle port (the reference is Python and cannot travel to the GPU box),
multi-threaded over element chunks, on a bounded sample of the same workload
(the config-5 rules on a 32x32x16 mesh), same steps / warm-up and the same
``config`` object as the GPU arm.  It never loads the product library.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 DoF/s per time step (LSRK & ADER) at 1/2/4/8 B200; % of roofline"
# LSRK: 32 B/DoF per stage (read u, r; write u, r), minus the r read of the
# first stage (a = 0) and the r store of the last (dead): SURVEY §8d's 160
# B/DoF per LSRK45 step counts the latter, the kernels no longer move it
BYTES_PER_DOF = {"lsrk45": 144.0, "lsrk59": 272.0, "ader_hdg": 48.0, "ader": 40.0}
STAGE_BYTES = 32.0   # per DoF per LSRK stage launch: read u, r; write u, r
# config 3 (curved, k=5): ADER-HDG 48 B/DoF of vectors + the per-point metric
# per K application (28.0 B/DoF) and the reduced-degree TCK metric (5.3 B/DoF)
CURVED_ADER_HDG_BYTES = 109.3
REF_SCALE = 0.25     # reference-arm sample: config rules on 1/4 of the elements per axis
DEFAULT_SCHEME = {"c1": "lsrk45", "c2": "lsrk45", "c3": "ader_hdg", "c4": "ader_hdg",
                  "c5": "lsrk45"}
NCU_METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
               "sm__sass_thread_inst_executed_op_dfma_pred_on.sum,"
               "sm__sass_thread_inst_executed_op_dmul_pred_on.sum,"
               "sm__sass_thread_inst_executed_op_dadd_pred_on.sum,"
               "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    """HBM: MEASURED_PEAKS.json (driver-written) else the profiling recipe's
    fallback; FP64: the DFMA microbenchmark (tools/fp64_peak.cu) committed
    under profiles/."""
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
            src = "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    fp64 = 34.2
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.jsonl")) as f:
            vals = [json.loads(line) for line in f if line.strip()]
        fp64 = max(v["tflops"] for v in vals if v.get("kind") == "dfma")
    except Exception:
        pass
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
# the workload description shared by both arms (same ``config`` object)

def workload_config(name, scheme, world):
    """The BASELINE config as a plain description (no product import)."""
    desc = {
        "c1": (256, 3, 2, "2D 16^2 periodic quad mesh, k=3, rho=c=1, standing mode"),
        "c2": (32768, 4, 3, "3D 32^3 periodic hex mesh, k=4, rho=c=1, seeded Fourier p"),
        "c3": (32768, 5, 3, "3D 32^3 hex mesh, degree-5 sin map, per-cell rho,c~U(0.5,2) "
                            "seed 1, Gaussian pulse"),
        "c4": (110592, 7, 3, "3D 48^3 periodic hex mesh, k=7, two-layer material, "
                             "seeded Fourier p"),
        "c5": (1048576, 4, 3, "3D 128x128x64 periodic hex mesh, k=4, per-cell rho,c~U(0.5,2) "
                              "seed 7, seeded Fourier p"),
    }[name]
    E, k, d = desc[0], desc[1], desc[2]
    dofs = E * (d + 1) * (k + 1) ** d
    return {"workload": f"{name}: {desc[3]}, {scheme}", "scheme": scheme, "elements": E,
            "degree": k, "dofs": dofs,
            "parallelism": "single GPU" if world == 1 else f"{world} x-slabs (one per GPU)",
            "l2": f"inputs larger than L2 (3 state vectors of {dofs * 8 / world / 1e6:.0f} MB "
                  "per GPU vs 126 MB L2); no flush" if dofs * 8 / world > 126e6 else
                  "state fits in L2 (small config)"}


# ---------------------------------------------------------------------------
# CPU arm: the oracle port of the reference algorithm on the host cores

def _oracle_problem(name, scale):
    """(problem, oracle operator) of config ``name`` at ``scale`` -- host-side
    input generation (numpy) + the oracle; no product library is loaded."""
    import oracle
    from paper_1805_03981_b200 import configs
    prob = configs.config(name, scale=scale, geometry="none")
    m = prob.mesh
    om = oracle.OracleMesh(m.d, m.n_per_dim, m.vertices, m.elements, m.neighbors,
                           m.boundary_kind)
    if name == "c3":
        base = oracle.build_cartesian(m.n_per_dim, 3, "periodic")
        geo = oracle.precompute_geometry(base, prob.k, g=5, mapping=configs.c3_mapping)
    else:
        geo = oracle.precompute_geometry(om, prob.k)
    op = oracle.OracleOperator(om, geo, oracle.OracleMaterial(prob.material.c,
                                                              prob.material.rho))
    return prob, om, op


def cpu_steps(name, scheme, scale, warmup, steps, max_wall=None):
    """Time the oracle on the config-``name`` rules at ``scale``: returns
    (DoF/s, threads, sample description, ms per sample step)."""
    from threadpoolctl import threadpool_limits
    from oracle import stepping as OS
    from oracle.parallel import ThreadedOracle
    with threadpool_limits(1):
        prob, om, op = _oracle_problem(name, scale)
        cr = prob.schemes.get(scheme, (0.2, 1))[0]
        dt = OS.compute_dt(cr, om, prob.material, prob.k)
        threads = os.cpu_count() or 1
        th = None
        if scheme.startswith("lsrk"):
            th = ThreadedOracle(op, threads)
            coeffs = OS.LSRK45 if scheme == "lsrk45" else OS.LSRK59
            step = lambda u: th.lsrk_step(u, dt, coeffs)
        else:
            threads = 1
            step = lambda u: OS.ader_step(u, dt, op, scheme)
        u = prob.state
        for _ in range(warmup):
            u = step(u)
        done, t0 = 0, time.perf_counter()
        while done < steps:
            u = step(u)
            done += 1
            if max_wall is not None and time.perf_counter() - t0 > max_wall:
                break
        wall = time.perf_counter() - t0
        if th is not None:
            th.close()
    m = prob.mesh
    sample = (f"{name} rules on {'x'.join(str(v) for v in m.n_per_dim)} "
              f"({m.n_elements} elements, k={prob.k}, {prob.dofs} DoF), {scheme}, "
              f"{done} steps in {wall:.1f} s, oracle port ({'threaded' if threads > 1 else 'scalar'})")
    return prob.dofs * done / wall, threads, sample, 1e3 * wall / done


def run_reference(args, rank, world):
    """``--impl reference``: rank 0 alone, the same config / steps / warm-up."""
    if rank != 0:
        return
    value, threads, sample, ms = cpu_steps(args.config, args.scheme, REF_SCALE, args.warmup,
                                           args.steps)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DoF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE rules)",
        "ms_per_step_note": "per step of the CPU sample (see cpu_baseline.sample)",
        "config": workload_config(args.config, args.scheme, world),
        "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# ncu probe: DRAM traffic and executed FP64 work of the dominant kernels,
# measured in this run on the same workload (a separate process under ncu;
# nothing it prints is a bench value)

def probe_main(args):
    """Run under ncu: one eager warm-up step, then one step whose launches ncu
    captures.  The state is device-random (instruction counts and DRAM bytes
    do not depend on the values), so no host-side state build is needed."""
    import torch
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import configs
    prob = configs.config(args.config, geometry="device", state=False)
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    shape = (prob.mesh.n_elements, prob.mesh.d + 1) + (prob.k + 1,) * prob.mesh.d
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
    cr = prob.schemes.get(args.scheme, (0.1, 1))[0]
    dt = W.compute_dt(cr, prob.mesh, prob.material, prob.k)
    st = W.make_stepper(W.SchemeConfig(scheme=args.scheme), op)
    st.use_graph = False
    for _ in range(2):
        res = st.run(u, dt, 1)
        if res is not u:
            u.copy_(res)
    torch.cuda.synchronize()


def ncu_probe(config, scheme, timeout=600):
    """Per-launch ncu metrics of one step's kernels (list of dicts) or None."""
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    lps = 5 if scheme == "lsrk45" else (9 if scheme == "lsrk59" else 2)
    with tempfile.TemporaryDirectory() as tmp:
        log = os.path.join(tmp, "ncu.csv")
        cmd = [ncu, "--metrics", NCU_METRICS, "--clock-control", "none", "--csv",
               "--log-file", log, "-k", "regex:stream|group|stage|curved|ader",
               "--launch-skip", str(lps), "--launch-count", str(lps),
               sys.executable, os.path.join(ROOT, "bench.py"), "--probe",
               "--config", config, "--scheme", scheme]
        try:
            p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        except Exception as exc:
            return None, f"ncu failed: {exc}"
        if p.returncode != 0 or not os.path.exists(log):
            return None, f"ncu rc {p.returncode}: {(p.stderr or p.stdout)[-300:]}"
        with open(log) as f:
            text = f.read()
    start = text.find('"ID"')
    if start < 0:
        return None, "no ncu rows"
    launches = {}
    for row in csv.DictReader(io.StringIO(text[start:])):
        key = int(row["ID"])
        rec = launches.setdefault(key, {"kernel": row["Kernel Name"].split("(")[0]})
        val = row["Metric Value"].replace(",", "")
        unit = row.get("Metric Unit", "")
        try:
            v = float(val)
        except ValueError:
            continue
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                 "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1.0)
        rec[row["Metric Name"]] = v * scale
    out = []
    for key in sorted(launches):
        r = launches[key]
        out.append({
            "kernel": r["kernel"],
            "ncu_s": r.get("gpu__time_duration.sum"),
            "dram_bytes": r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0),
            "dram_read": r.get("dram__bytes_read.sum"),
            "dram_write": r.get("dram__bytes_write.sum"),
            "fp64_flops": 2 * r.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
                          + r.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0)
                          + r.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0),
            "fp64_pipe_pct": r.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        })
    return out, "ok"


# ---------------------------------------------------------------------------
# GPU arm, one GPU

def _timed(torch, fn, repeats, stream):
    """Median over ``repeats`` of the CUDA-event time of fn() (ms)."""
    times = []
    for _ in range(repeats):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return statistics.median(times), times


def measure_configs(torch, W, hbm, fp64, skip):
    """ms/step and DoF/s of the other BASELINE configs / schemes on this GPU
    (device-resident state, CUDA-graph replay, CUDA events; median of 3)."""
    from paper_1805_03981_b200 import configs
    plan = [("c1", "lsrk45", 10), ("c2", "lsrk45", 100), ("c2", "ader_hdg", 100),
            ("c3", "ader_hdg", 50), ("c3", "lsrk45", 50),
            ("c4", "ader_hdg", 20), ("c4", "lsrk45", 20)]
    out, cache = {}, {}
    for cfg, scheme, steps in plan:
        if (cfg, scheme) in skip:
            continue
        try:
            t0 = time.perf_counter()
            if cfg not in cache:
                cache.clear()
                torch.cuda.empty_cache()
                prob = configs.config(cfg, geometry="device")
                op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
                cache[cfg] = (prob, op, time.perf_counter() - t0)
            prob, op, setup_s = cache[cfg]
            cr = prob.schemes.get(scheme, (0.1, 1))[0]
            dt = W.compute_dt(cr, prob.mesh, prob.material, prob.k)
            st = W.make_stepper(W.SchemeConfig(scheme=scheme, courant=cr), op)
            u = torch.from_numpy(prob.state).cuda()
            st.run(u, dt, 6)                      # warm-up + graph capture
            s = torch.cuda.current_stream()
            ms, _ = _timed(torch, lambda: st.run(u, dt, steps), 3, s)
            ms /= steps
            bpd = BYTES_PER_DOF.get(scheme, 0.0)
            if cfg == "c3" and scheme == "ader_hdg":
                bpd = CURVED_ADER_HDG_BYTES
            out[f"{cfg}_{scheme}"] = {
                "ms_per_step": ms, "dofs_per_s": prob.dofs / (ms * 1e-3), "dofs": prob.dofs,
                "steps": steps, "courant": cr, "setup_s": setup_s,
                "hbm_algorithmic_gbs": bpd * prob.dofs / ms / 1e6,
                "hbm_frac": bpd * prob.dofs / ms / 1e6 / hbm,
                "bytes_per_dof": bpd, "finite": bool(torch.isfinite(u).all()),
                "workload": prob.description}
            del u, st
        except Exception as exc:                   # reported, not fatal
            out[f"{cfg}_{scheme}"] = {"error": str(exc)[:200]}
    cache.clear()
    torch.cuda.empty_cache()
    return out


def run_single(args):
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import _lib, configs
    from paper_1805_03981_b200._lib import check, lib

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    hbm, hbm_src, fp64_peak = peaks()
    t_setup = time.perf_counter()
    prob = configs.config(args.config, geometry="device")
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    setup_s = time.perf_counter() - t_setup
    scheme = args.scheme
    cr = prob.schemes.get(scheme, (0.2, 1))[0]
    dt = W.compute_dt(cr, prob.mesh, prob.material, prob.k)
    dofs = prob.dofs
    state_bytes = dofs * 8
    host = torch.from_numpy(prob.state).pin_memory()
    u = host.to(dev)
    stepper = W.make_stepper(W.SchemeConfig(scheme=scheme, courant=cr), op)
    s = torch.cuda.current_stream()
    sp = op.stream

    # warm-up (eager W steps, then the CUDA graph of the production path)
    res = stepper.run(u, dt, args.warmup)
    if res is not u:
        u.copy_(res)
    stepper.capture(u, dt)
    torch.cuda.synchronize()

    # timed region: exactly K steps of the production path, R repeats, median
    n_launch = args.steps * stepper.launches_per_step()
    with ClockSampler(dev.index or 0) as clk:
        total_ms, all_ms = _timed(torch, lambda: stepper.run(u, dt, args.steps),
                                  args.repeats, s)
    assert bool(torch.isfinite(u).all())
    ms_step = total_ms / args.steps
    value = dofs * args.steps / (total_ms * 1e-3)

    # per-launch durations of the dominant kernel (CUDA events around every
    # launch, on the stream the kernels run on) in an instrumented eager pass
    b1, b2 = stepper.buffers(u)
    roof, kern = {}, {}
    if scheme.startswith("lsrk"):
        coeffs = W.LSRK45 if scheme == "lsrk45" else W.LSRK59
        evs, nbytes = [], []
        cur, nxt, r = u, b1, b2
        for _ in range(args.steps):
            for i, (a, b) in enumerate(zip(coeffs.a, coeffs.b)):
                last = i == coeffs.stages - 1        # as DeviceStepper: r dead after it
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                check(lib().wk_lsrk_stage_ex(op._ctx, op._ptr(cur), op._ptr(nxt), op._ptr(r),
                                             float(a), float(b), float(dt), int(last), sp))
                e1.record(s)
                evs.append((e0, e1, a != 0.0 and not last))
                cur, nxt = nxt, cur
        torch.cuda.synchronize()
        ms_all = [x.elapsed_time(y) for x, y, _ in evs]
        ms_full = [m for m, (_, _, full) in zip(ms_all, evs) if full]   # middle stages
        avg = statistics.mean(ms_full)
        achieved = STAGE_BYTES * dofs / (avg * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None,
                "kernel": "LSRK stage kernel (the middle stages; the first reads no r and "
                          "the last stores none: 24 B/DoF each, 144 B/DoF per LSRK45 step)",
                "peak_source": hbm_src, "avg_launch_ms": avg,
                "algorithmic_bytes": f"32 B/DoF x {dofs} DoF = {STAGE_BYTES * dofs / 1e9:.3f} GB "
                                     "per stage launch (read u, r; write u, r; SURVEY 8d)",
                "timing": "CUDA events around every launch in an eager pass of the same K "
                          "steps (the timed region replays the CUDA graph)",
                "step_share": sum(ms_all) / args.steps / ms_step}
    if hasattr(stepper, "_graph"):
        stepper._graph = None

    # end to end through the public API: pinned host StateVector in, K steps
    # on the device, state back to host (one H2D + K steps + one D2H)
    st_host = W.StateVector(host.numpy(), prob.k, prob.mesh.d)
    W.advance(st_host, dt, 3 * stepper.GRAPH_STEPS, stepper)   # warm-up incl. graph
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(args.repeats):
        t0 = time.perf_counter()
        out = W.advance(st_host, dt, args.steps, stepper)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e_t)
    assert np.all(np.isfinite(out.data[:8]))
    del out
    e2e = {"value": dofs * args.steps / e2e_s, "unit": "DoF/s",
           "h2d_bytes_per_step": state_bytes / args.steps,
           "d2h_bytes_per_step": state_bytes / args.steps,
           "api": "paper_1805_03981_b200.advance(StateVector(pinned numpy), dt, K, "
                  "make_stepper(...)): one H2D of the state, K steps, one D2H "
                  "(host wall clock, median of R)"}

    extras = {}
    if not args.no_extras and scheme.startswith("lsrk"):
        # ADER-HDG order k+1 on the same mesh and state: the metric's "ADER" half
        sta = W.make_stepper(W.SchemeConfig(scheme="ader_hdg"), op)
        cra = prob.schemes.get("ader_hdg", (0.1, 1))[0]
        dta = W.compute_dt(cra, prob.mesh, prob.material, prob.k)
        ua = host.to(dev)
        sta.run(ua, dta, max(args.warmup, 6))
        torch.cuda.synchronize()
        ms_a, _ = _timed(torch, lambda: sta.run(ua, dta, args.steps), args.repeats, s)
        ms_a /= args.steps
        variant, pol = _lib.WK_ADER_HDG, _lib.POLICY["every_second"]
        V, Y = sta.buffers(ua)
        evs = []
        for _ in range(args.steps):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(s)
            check(lib().wk_ader_a(op._ctx, variant, pol, op._ptr(ua), op._ptr(V), op._ptr(Y),
                                  float(dta), sp))
            e[1].record(s)
            check(lib().wk_ader_b(op._ctx, variant, op._ptr(ua), op._ptr(V), op._ptr(Y), sp))
            e[2].record(s)
            evs.append(e)
        torch.cuda.synchronize()
        ka = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
        kb = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
        extras["ader_hdg"] = {
            "value": dofs / (ms_a * 1e-3), "unit": "DoF/s", "ms_per_step": ms_a,
            "steps": args.steps, "courant": cra,
            "kernel_a_ms": ka, "kernel_b_ms": kb,
            "hbm_frac_step": 48.0 * dofs / (ms_a * 1e-3) / 1e9 / hbm,
            "note": "ADER-HDG order k+1, every_second reduction, same mesh/state; kernel A "
                    "(W = M^-1 K U, V, Taylor loop) is FP64-bound, kernel B (M^-1 K y "
                    "update) HBM-bound"}
        kern = {"ka": ka, "kb": kb}
        del ua, sta

    # DRAM traffic + executed FP64 work of the same kernels, measured in this
    # run by ncu on the same workload (separate process; timings not used)
    if not args.no_probe:
        del u
        torch.cuda.empty_cache()
        rows, msg = ncu_probe(args.config, scheme)
        if rows:
            full = [r for r in rows if r["dram_bytes"]]
            if scheme.startswith("lsrk") and len(full) >= 2:
                mid = full[1:-1] if len(full) >= 3 else full[1:]     # the 32 B/DoF launches
                per = statistics.mean(r["dram_bytes"] for r in mid)
                roof["traffic"] = per
                roof["traffic_over_algorithmic"] = per / (STAGE_BYTES * dofs)
                roof["fp64_pipe_pct"] = statistics.mean(r["fp64_pipe_pct"] or 0 for r in mid)
            roof["ncu"] = {"launches": rows, "source": "ncu --metrics (this run, one step after "
                           "one warm-up step, device-random state; profiler times not used)"}
        else:
            roof["ncu"] = {"error": msg}
        if "ader_hdg" in extras:
            rows_a, msg_a = ncu_probe(args.config, "ader_hdg")
            if rows_a and len(rows_a) >= 2:
                A, B = rows_a[0], rows_a[1]
                fa = A["fp64_flops"] / (kern["ka"] * 1e-3) / 1e12
                extras["ader_hdg"]["roofline"] = {
                    "bound": "fp64", "kernel": "ADER kernel A (" + A["kernel"] + ")",
                    "achieved": fa, "peak": fp64_peak, "unit": "TFLOP/s", "frac": fa / fp64_peak,
                    "executed_flops": A["fp64_flops"],
                    "flops": "executed FP64 (ncu: 2 DFMA + DMUL + DADD thread instructions "
                             "per launch) / event-timed launch duration",
                    "peak_source": "DFMA microbenchmark (profiles/fp64_peak_r01.jsonl)",
                    "fp64_pipe_pct": A["fp64_pipe_pct"],
                    "traffic": A["dram_bytes"], "algorithmic_bytes": 24.0 * dofs,
                    "hbm_frac": 24.0 * dofs / (kern["ka"] * 1e-3) / 1e9 / hbm}
                extras["ader_hdg"]["kernel_b_roofline"] = {
                    "bound": "hbm", "kernel": B["kernel"],
                    "achieved": 24.0 * dofs / (kern["kb"] * 1e-3) / 1e9, "peak": hbm,
                    "unit": "GB/s", "frac": 24.0 * dofs / (kern["kb"] * 1e-3) / 1e9 / hbm,
                    "traffic": B["dram_bytes"], "fp64_pipe_pct": B["fp64_pipe_pct"],
                    "algorithmic_bytes": "24 B/DoF (read U, V, y; write U)"}
            else:
                extras["ader_hdg"]["roofline"] = {"error": msg_a}
    else:
        del u

    if not args.no_extras and not args.no_configs:
        extras["configs"] = measure_configs(torch, W, hbm, fp64_peak,
                                            skip={(args.config, scheme)})

    cpu = None
    if not args.no_cpu_baseline:
        try:
            v, threads, sample, _ = cpu_steps(args.config, scheme, REF_SCALE, 1, 5, max_wall=25)
            cpu = {"value": v, "unit": "DoF/s", "cores": threads, "kind": "port",
                   "sample": sample}
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": "DoF/s", "cores": 0, "kind": "port",
                   "sample": f"failed: {exc}"}

    line = {
        "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "repeats_ms": all_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Fourier-mode pressure, BASELINE rules)",
        "config": workload_config(args.config, scheme, 1),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": n_launch,
        "clocks": clk.summary(), "fp64_peak_tflops": fp64_peak, "setup_s": setup_s,
    }
    line.update(extras)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def spawn_torchrun(argv, n):
    """--gpus N > 1 outside torchrun: relaunch this script under torchrun."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    port = env.get("MASTER_PORT", "29541")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", port,
           os.path.abspath(__file__)] + argv
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--scheme", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config table (configs 1-4, both schemes)")
    ap.add_argument("--no-probe", action="store_true", help="skip the ncu traffic/FP64 probe")
    ap.add_argument("--probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--slab-path", action="store_true",
                    help="run the multi-GPU slab bench even at WORLD_SIZE=1 (path check)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.scheme is None:
        args.scheme = DEFAULT_SCHEME[args.config]
    if args.probe:
        probe_main(args)
        return
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, max(world, args.gpus))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "n_gpus": args.gpus, "error":
                              f"--gpus {args.gpus} requested, {have} visible"}), flush=True)
            sys.exit(1)
        sys.exit(spawn_torchrun(sys.argv[1:], args.gpus))
    if world > 1 or args.slab_path:
        from paper_1805_03981_b200 import slabs
        if "RANK" not in os.environ:   # --slab-path without torchrun: a one-rank job
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0",
                              MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29533"))
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        hbm, hbm_src, _ = peaks()
        slabs.bench_main(args, rank, world, local, METRIC, clock_sampler=ClockSampler,
                         hbm_peak=hbm, hbm_src=hbm_src,
                         config=workload_config(args.config, args.scheme, world))
        return
    run_single(args)


if __name__ == "__main__":
    main()
