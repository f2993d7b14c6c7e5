"""Stepper-state regressions of the device stepper (round-1 advisor findings).

* ``advance`` / the ``(state, dt)`` closure must return a FRESH state every
  call, as the reference does (stepping.py:305-308): with the odd-stage
  LSRK45 an odd step count used to end in the stepper's ping-pong buffer,
  which the next call overwrote.
* A CUDA graph captured for one dt must keep that dt's Taylor weights when
  the same stepper runs eagerly with another dt in between (the weights used
  to live in one device buffer per TCK program, rewritten per dt).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _problem():
    from paper_1805_03981_b200 import configs
    return configs.config("c2", scale=0.125)        # 4^3 periodic k=4


def test_consecutive_single_steps_do_not_alias(cuda):
    import paper_1805_03981_b200 as W
    prob = _problem()
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    step = W.make_stepper(W.SchemeConfig(scheme="lsrk45"), op)
    dt = W.compute_dt(0.2, prob.mesh, prob.material, prob.k)
    s0 = W.StateVector(torch.from_numpy(prob.state).to(cuda), prob.k, 3)
    s1 = step(s0, dt)
    keep = s1.data.clone()
    s2 = step(s1, dt)
    assert s1.data.data_ptr() != s2.data.data_ptr()
    assert torch.equal(s1.data, keep)
    assert not torch.equal(s2.data, keep)
    # and the pair equals two steps taken at once
    s2b = W.advance(s0, dt, 2, step)
    assert torch.equal(s2.data, s2b.data)


@pytest.mark.parametrize("scheme,reduction", [("ader_hdg", "every_second"),
                                              ("ader_hdg", "every_step"),
                                              ("ader", "none")])
def test_graph_keeps_its_dt_after_eager_run_with_other_dt(cuda, scheme, reduction):
    import paper_1805_03981_b200 as W
    prob = _problem()
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    cfg = W.SchemeConfig(scheme=scheme, degree_reduction=reduction)
    dt1 = W.compute_dt(0.1, prob.mesh, prob.material, prob.k)
    dt2 = 0.5 * dt1
    u0 = torch.from_numpy(prob.state).to(cuda)

    st = W.make_stepper(cfg, op)
    u = u0.clone()
    st.run(u, dt1, 8)                    # eager warm-up + graph of dt1
    v = u0.clone()
    st.run(v, dt2, 1)                    # eager with another dt (rewrote weights before)
    u.copy_(u0)
    res = st.run(u, dt1, 8)              # replays the dt1 graph
    assert res is u

    ref = W.make_stepper(cfg, op)
    ref.use_graph = False
    w = u0.clone()
    ref.run(w, dt1, 8)
    assert torch.equal(u, w)
    assert np.isfinite(u.cpu().numpy()).all()


@pytest.mark.parametrize("cfg,scale", [("c2", 0.25), ("c4", 1.0 / 12), ("c3", 0.125)])
def test_last_stage_without_r_store(cuda, cfg, scale):
    """wk_lsrk_stage_ex(r_dead=1) -- the last stage of a step, whose register
    no later stage reads (stepping.py:184-195 allocates r per step) -- must
    give the same new state as the plain stage, bit for bit; the stepper's
    trajectory then equals plain stage launches."""
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import configs
    from paper_1805_03981_b200._lib import check, lib
    prob = configs.config(cfg, scale=scale) if cfg != "c3" else \
        configs.config(cfg, scale=scale, geometry="device")
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    dt = W.compute_dt(0.2, prob.mesh, prob.material, prob.k)
    u = torch.from_numpy(prob.state).to(cuda)
    r0 = torch.randn_like(u)
    a, b = W.LSRK45.a[-1], W.LSRK45.b[-1]
    outs = []
    for dead in (0, 1):
        r = r0.clone()
        out = torch.empty_like(u)
        check(lib().wk_lsrk_stage_ex(op._ctx, op._ptr(u), op._ptr(out), op._ptr(r), float(a),
                                     float(b), float(dt), dead, op.stream))
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    # two steps through the stepper (last stages with r_dead) == plain stages
    cur, nxt, r = u.clone(), torch.empty_like(u), torch.empty_like(u)
    for _ in range(2):
        for a, b in zip(W.LSRK45.a, W.LSRK45.b):
            check(lib().wk_lsrk_stage(op._ctx, op._ptr(cur), op._ptr(nxt), op._ptr(r), float(a),
                                      float(b), float(dt), op.stream))
            cur, nxt = nxt, cur
    torch.cuda.synchronize()
    if not getattr(op, "small_run", False):
        got = W.advance(W.StateVector(u.clone(), prob.k, 3), dt, 2,
                        W.make_stepper(W.SchemeConfig(scheme="lsrk45"), op)).data
        assert torch.equal(got, cur)


def test_one_group_kernel_matches_direction_parallel(cuda):
    """WK_STREAM=seq (the one-group stage kernel, the fallback of DESIGN.md §6)
    and the default direction-parallel kernel share the arithmetic -- same
    expressions, p = (P_0 + P_1) + P_2 -- so two LSRK45 steps and one ADER-HDG
    step agree bit for bit.  The selection is read once per process, hence the
    subprocess."""
    import hashlib
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, hashlib, torch; sys.path.insert(0, %r)\n"
        "import paper_1805_03981_b200 as W\n"
        "from paper_1805_03981_b200 import configs\n"
        "p = configs.config('c2', scale=0.25)\n"
        "op = W.AcousticOperator(p.mesh, p.geometry, p.material)\n"
        "dt = W.compute_dt(0.2, p.mesh, p.material, p.k)\n"
        "s = W.StateVector(torch.from_numpy(p.state).cuda(), p.k, 3)\n"
        "a = W.advance(s, dt, 2, W.make_stepper(W.SchemeConfig(scheme='lsrk45'), op)).data\n"
        "b = W.ader_step(s, dt, op, 'ader_hdg').data\n"
        "print(hashlib.sha256(a.cpu().numpy().tobytes() + b.cpu().numpy().tobytes()).hexdigest())\n"
    ) % root
    out = {}
    for mode in ("seq", "dir"):
        env = dict(os.environ, WK_STREAM=mode, WK_SMALL="0")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = r.stdout.strip().splitlines()[-1]
    assert out["seq"] == out["dir"]
