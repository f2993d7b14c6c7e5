"""Cost model, kernel-call counter emulation and CLI plumbing (CPU).

Pinned to tests/golden/cost.json, made by running the unmodified reference
(tests/golden/make_golden_cost.py): kernels.py:191-342 model numbers, the
reference operator's KernelCounter tallies per method, the reference
``opcount`` table (cli.py:247-276)."""

from __future__ import annotations

import contextlib
import io
import json
import os

import pytest

from paper_1805_03981_b200 import cli, cost

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cost.json")))
POLICIES = ("none", "every_step", "every_second", "every_third")


@pytest.mark.parametrize("key", sorted(GOLD["model"]))
def test_model_matches_reference(key):
    d, k = (int(v) for v in key.split("_"))
    g = GOLD["model"][key]
    assert cost.kernel_call_table(k, d) == g["table"]
    for s, ref in g["schemes"].items():
        rep = cost.scheme_cost(k, d, s)
        assert {f: getattr(rep, f) for f in ref} == ref, s
    for p, ref in g["tck"].items():
        assert cost.tck_cost_model(k, d, p) == ref, p


def test_model_errors():
    with pytest.raises(ValueError):
        cost.cost_tensorial(0, 3)
    with pytest.raises(ValueError):
        cost.kernel_call_table(3, 4)
    with pytest.raises(ValueError):
        cost.scheme_cost(3, 3, "euler")
    with pytest.raises(ValueError):
        cost.scheme_cost(3, 3, "rk")
    assert cost.scheme_cost(3, 3, "rk", stages=5).c_scheme_total == \
        cost.scheme_cost(3, 3, "lsrk45").c_scheme_total


def _emulate(name, E, d, k):
    c = cost.KernelCounter()
    c.enabled = True
    kind, *rest = name.split(":")
    if kind == "apply_K":
        cost.count_apply_K(c, E, d, k, rest[0])
    elif kind in ("apply_inverse_mass", "apply_mass"):
        cost.count_mass(c, E, d, k)
    elif kind == "rhs":
        cost.count_apply_K(c, E, d, k)
        cost.count_mass(c, E, d, k)
    elif kind == "tck":
        cost.count_tck(c, E, d, k, rest[0], bool(int(rest[1])))
    elif kind == "step":
        cost.count_scheme_step(c, rest[0], E, d, k, rest[1])
    return c.counts


@pytest.mark.parametrize("case", range(len(GOLD["counts"])))
def test_counter_emulation_matches_reference_tallies(case):
    g = GOLD["counts"][case]
    for name, ref in g["calls"].items():
        assert _emulate(name, g["elements"], g["d"], g["k"]) == ref, name


def test_counter_interface():
    c = cost.KernelCounter()
    c.record("mass", units=3, n_out=4, n_in=4, lines=4)
    assert c.counts == {}                       # off by default
    c.enabled = True
    c.record("mass", units=3, n_out=4, n_in=4, lines=4)
    c.record("stiffness", units=2, n_out=4, n_in=4, lines=1, face=True)
    assert c.calls("mass") == 3 and c.calls("stiffness", face=True) == 2
    assert c.total_flops() == 3 * cost.kernel_flops(4, 4, 4) + 2 * cost.kernel_flops(4, 4, 1)
    other = cost.KernelCounter()
    other.enabled = True
    other.record("mass", units=1, n_out=4, n_in=4, lines=4)
    c.merge(other)
    assert c.calls("mass") == 4
    c.reset()
    assert c.total_flops() == 0


def test_opcount_table_matches_reference():
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert cli.main(["opcount"]) == 0
    assert buf.getvalue() == GOLD["opcount"]


def test_opcount_json(tmp_path):
    js = tmp_path / "o.json"
    with contextlib.redirect_stdout(io.StringIO()):
        assert cli.main(["opcount", "--json", str(js)]) == 0
    payload = json.loads(js.read_text())
    assert len(payload["records"]) == 2 * 12 * 2
    assert payload["records"][0]["command"] == "opcount"


@pytest.mark.parametrize("argv,msg", [
    (["run", "--degree", "0"], "degree must be at least 1"),
    (["run", "--dim", "4"], "invalid choice"),
    (["run", "--scheme", "euler"], "invalid choice"),
    (["run", "--deform", "0.7"], "deform amplitude"),
    (["run", "--tau", "-1"], "tau must be positive"),
    (["bogus"], "invalid choice"),
    (["run", "--degree", "9"], "degrees 1..8"),
])
def test_config_errors_exit_1(argv, msg, capsys):
    assert cli.main(argv) == cli.EXIT_CONFIG
    assert msg in capsys.readouterr().err


def test_config_file(tmp_path, capsys):
    cfg = tmp_path / "bench.cfg"
    cfg.write_text("turbo = on\n")
    assert cli.main(["run", "--config", str(cfg)]) == cli.EXIT_CONFIG
    assert "unknown key" in capsys.readouterr().err
    cfg.write_text("degree = x\n")
    assert cli.main(["run", "--config", str(cfg)]) == cli.EXIT_CONFIG
    assert "bad value" in capsys.readouterr().err
    cfg.write_text("degree 3\n")
    assert cli.main(["run", "--config", str(cfg)]) == cli.EXIT_CONFIG
    assert "KEY=VALUE" in capsys.readouterr().err


def test_config_resolution(tmp_path):
    cfg = tmp_path / "bench.cfg"
    cfg.write_text("degree = 3\nelements = 2\nscheme = ader\nend-time = 0.125\n"
                   "reduction = none  # trailing comment\nboundary = periodic\n")
    rc = cli.resolve(["run", "--config", str(cfg), "--elements", "4"])
    assert (rc.degree, rc.elements, rc.scheme, rc.end_time) == (3, 4, "ader", 0.125)
    assert (rc.reduction, rc.boundary, rc.device) == ("none", "periodic", "cuda")
    cfg.write_text("scheme = euler\n")
    with pytest.raises(cli.ConfigError):
        cli.resolve(["run", "--config", str(cfg)])
    for bad in (["run", "--dim", "4"], ["run", "--courant", "-1"], ["run", "--degree", "9"]):
        with pytest.raises(cli.ConfigError):
            cli.resolve(bad)
    assert cli.main(["run", "--levels", "0"]) == cli.EXIT_CONFIG


def test_model_flops_per_step_matches_reference_cli():
    for rec in GOLD["run"]:
        study = cli.Study(cli.resolve(rec["args"]))
        assert study.model_flops(study.s.elements) == rec["model_flops"]
        assert study.dofs(study.s.elements) == rec["dofs"]


@pytest.mark.parametrize("i", range(len(GOLD["hdg_flux"])))
def test_hdg_flux_matches_reference(i):
    """operator.hdg_flux (reference operator.py:70-87) on the reference's
    outputs, plus its swap antisymmetry (minus <-> plus with n -> -n negates)."""
    import numpy as np
    from paper_1805_03981_b200 import hdg_flux
    g = GOLD["hdg_flux"][i]
    a = lambda k: np.asarray(g[k])
    fv, fp = hdg_flux((a("vm"), a("pm")), (a("vp"), a("pp")), a("n"), g["c"], g["rho"], g["tau"])
    np.testing.assert_allclose(fv, a("fv"), rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(fp, a("fp"), rtol=1e-14, atol=1e-15)
    sv, sp = hdg_flux((a("vp"), a("pp")), (a("vm"), a("pm")), -a("n"), g["c"], g["rho"], g["tau"])
    np.testing.assert_allclose(sv, -fv, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(sp, -fp, rtol=1e-14, atol=1e-15)
