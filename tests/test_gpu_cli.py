"""The study harness on the GPU: reference CLI records
reproduced through the fused kernels, the counting-mode FLOP identity, and
the counter emulation of the GPU operator's methods (golden: reference runs
in tests/golden/cost.json, tests/golden/make_golden_cost.py)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_1805_03981_b200 import cli, cost

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cost.json")))


def _records(out):
    lines = out.strip().splitlines()
    head = lines[0].split(",")
    return [dict(zip(head, ln.split(","))) for ln in lines[1:]]


@pytest.mark.parametrize("i", range(len(GOLD["run"])))
def test_run_matches_reference_record(i, cuda, capsys):
    g = GOLD["run"][i]
    assert cli.main(g["args"]) == cli.EXIT_OK
    rec = _records(capsys.readouterr().out)[0]
    assert int(rec["steps"]) == g["steps"]
    assert int(rec["dofs"]) == g["dofs"] and int(rec["model_flops"]) == g["model_flops"]
    # the L2 error of the GPU trajectory equals the reference's: the states
    # agree to ~1e-14, far below the discretisation error being measured
    assert float(rec["l2_err"]) == pytest.approx(g["l2_err"], rel=1e-7)
    assert float(rec["wall_s"]) > 0 and float(rec["dofs_per_s"]) > 0


@pytest.mark.parametrize("scheme", ["ader", "ader-hdg", "lsrk45", "rk4"])
def test_throughput_counting_matches_model(scheme, cuda, tmp_path, capsys):
    js = tmp_path / "tp.json"
    assert cli.main(["throughput", "--degree", "3", "--elements", "4", "--scheme", scheme,
                     "--reduction", "none", "--json", str(js)]) == cli.EXIT_OK
    rec = _records(capsys.readouterr().out)[0]
    payload = json.loads(js.read_text())
    assert payload["counted_flops"] == int(rec["model_flops"])
    assert int(rec["steps"]) == 100 and float(rec["dofs_per_s"]) > 0


def test_throughput_3d_reduction(cuda, capsys):
    assert cli.main(["throughput", "--dim", "3", "--degree", "4", "--elements", "4",
                     "--scheme", "ader-hdg", "--boundary", "periodic"]) == cli.EXIT_OK
    rec = _records(capsys.readouterr().out)[0]
    assert int(rec["dofs"]) == 4 ** 3 * 4 * 125


def test_convergence_orders(cuda, tmp_path, capsys):
    js = tmp_path / "c.json"
    assert cli.main(["convergence", "--degree", "2", "--elements", "2", "--levels", "3",
                     "--scheme", "lsrk45", "--end-time", "0.25", "--json", str(js)]) == 0
    payload = json.loads(js.read_text())
    assert len(payload["records"]) == 3
    assert all(o > 2.0 for o in payload["observed_orders"])


def test_courant_2d(cuda, capsys):
    assert cli.main(["courant", "--degree", "2", "--elements", "2", "--scheme", "lsrk45",
                     "--boundary", "periodic"]) == cli.EXIT_OK
    rec = _records(capsys.readouterr().out)[0]
    assert 0.1 < float(rec["cr_crit"]) < 2.0


def test_numerical_guard_exit_2(cuda, capsys):
    assert cli.main(["run", "--degree", "3", "--elements", "4", "--scheme", "lsrk45",
                     "--courant", "5.0", "--end-time", "2.0"]) == cli.EXIT_NUMERICAL
    assert "numerical guard" in capsys.readouterr().err


def test_operator_counter_emulation(cuda):
    """The GPU operator's methods and fused steppers tally what the reference
    operator records for the same calls (golden per-method tallies)."""
    import torch
    import paper_1805_03981_b200 as W
    for g in GOLD["counts"]:
        d, k = g["d"], g["k"]
        n = round(g["elements"] ** (1.0 / d))
        mesh = W.build_cartesian(n, d, "periodic")
        if g["deform"]:
            mesh = W.deform(mesh, g["deform"])
        mat = W.Material.uniform(mesh)
        degs = sorted(set(sum((cost.reduction_degrees(k, p) for p in
                               ("none", "every_step", "every_second", "every_third")), ())))
        geo = W.precompute_geometry(mesh, k, reduced_degrees=tuple(degs), device="cuda")
        op = W.AcousticOperator(mesh, geo, mat)
        st = W.initial_state(mesh, k, mat, m=1)
        c = op.counter
        for name, ref in g["calls"].items():
            kind, *rest = name.split(":")
            c.reset()
            c.enabled = True
            if kind == "apply_K":
                op.apply_K(st, rest[0])
            elif kind == "apply_inverse_mass":
                op.apply_inverse_mass(st)
            elif kind == "apply_mass":
                op.apply_mass(st)
            elif kind == "rhs":
                op.rhs(st)
            elif kind == "tck":
                W.tck_evaluate(st, 1e-3, op, rest[0], shift=bool(int(rest[1])))
            elif kind == "step":
                step = W.make_stepper(W.SchemeConfig(scheme=rest[0], degree_reduction=rest[1]), op)
                step(W.StateVector(st.data.clone(), k, d), 1e-3)
            c.enabled = False
            torch.cuda.synchronize()
            assert c.counts == ref, (g["d"], g["k"], name)
